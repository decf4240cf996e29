"""Small sageattn invocations for compute-sanitizer (racecheck / synccheck / memcheck / initcheck).

Covers head dims 32 / 64 / 96 / 128 (32 and 96 zero-padded onto the 64 / 128 kernels), causal and non-causal, a ragged tail (N % 64 != 0 and N % 128 != 0),
GQA, FP16 and FP32 PV accumulation and the instrumented (RunReport) kernel variant, at small
B*H so the sanitizer's serialisation stays within minutes.  Exits non-zero on a CUDA error.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py

Run memcheck/initcheck with PYTORCH_NO_CUDA_MEMORY_CACHING=1 so every tensor is its own allocation
and an out-of-bounds access past a tensor's end is reported (tools/gpu_sanitize.sh does).
"""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_2505_21136_b200 as sa  # noqa: E402

CASES = [
    # (B, Hq, Hkv, N, D, causal, pv_accum)
    (1, 2, 2, 1000, 128, False, "fp16"),
    (1, 2, 2, 1000, 128, True, "fp16"),
    (1, 2, 1, 777, 64, False, "fp16"),
    (1, 2, 2, 777, 64, True, "fp16"),
    (1, 1, 1, 1100, 128, False, "fp32"),
    (1, 1, 1, 17776 // 8, 64, False, "fp16"),  # the CogVideoX ragged tail (48 real keys in the last block)
    (1, 2, 2, 640, 128, False, "fp16-depth1"),  # buffering depth 1: each k=32 group its own FP16 accumulation
    (1, 2, 1, 333, 32, True, "fp16"),   # head_dim 32 on the 64 kernel: padded-channel loads and stores
    (1, 2, 2, 1000, 96, False, "fp16"),  # head_dim 96 on the 128 kernel
]


def main() -> None:
    g = torch.Generator(device="cuda").manual_seed(0)
    only = sys.argv[1] if len(sys.argv) > 1 else None
    for i, (B, Hq, Hkv, N, D, causal, acc) in enumerate(CASES):
        if only is not None and str(i) != only:
            continue
        q = torch.randn(B, Hq, N, D, device="cuda", dtype=torch.bfloat16, generator=g)
        k = torch.randn(B, Hkv, N, D, device="cuda", dtype=torch.bfloat16, generator=g)
        v = torch.randn(B, Hkv, N, D, device="cuda", dtype=torch.bfloat16, generator=g)
        kw = dict(pv_accum="fp16", buffering_depth=1) if acc == "fp16-depth1" else dict(pv_accum=acc)
        o = sa.sageattn(q, k, v, "HND", causal, None, **kw)
        rep = sa.new_report("cuda")
        o2 = sa.sageattn(q, k, v, "HND", causal, None, report=rep, **kw)
        torch.cuda.synchronize()
        ok = torch.equal(o, o2)
        print(f"case {i}: B={B} Hq={Hq} Hkv={Hkv} N={N} D={D} causal={causal} acc={acc} "
              f"finite={bool(torch.isfinite(o).all())} instr==plain={ok}", flush=True)
        if not ok:
            raise SystemExit("instrumented kernel differs from the production kernel")


if __name__ == "__main__":
    main()
