"""B200 range sweep: the reference's `lpattn sweep --preset table2` (cli.py:225-310) on the GPU.

For every (P_r, V_r, depth) pair of the sweep, on the same deterministic inputs, run the sm_100a path
through `attention_quantized` and compare it with exact FP64 attention (computed on the GPU in
float64, the role of attention_reference, attention.py:186-220).  Rows carry the reference's
REPORT_FIELDS (cli.py:34-57) so the CSV is interchangeable with the reference's; `wall_time` is
the GPU call's wall time.

    python -m paper_2505_21136_b200.sweep --preset table2 --heads 8 --seq-len 1024 --head-dim 128

This reproduces the paper's Table-2 invariance and the reference's acceptance
check c06 (tests/test_acceptance.py:187-220): cossim >= 0.999 for every pair, pairwise
|d cossim| <= 1e-3 and |d L1| <= 2e-4, including the FP32-accumulator SageAttention2 baseline
(448, 448, depth 1, overflow waived).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

from .api import attention_quantized, compare
from .config import AttentionConfig, RangeConfig, RangeConfigError

# cli.py:59
TABLE2_PAIRS = [(448.0, 2.25, 2), (224.0, 4.5, 2), (112.0, 9.0, 2)]
# the SageAttention2 baseline the acceptance test compares against (tests/test_acceptance.py:201-205)
FP32_BASELINE = (448.0, 448.0, 1)

REPORT_FIELDS = [
    "seq_len", "head_dim", "heads", "block_q", "block_k", "qk_bits", "p_r", "v_r", "depth", "causal",
    "smoothing", "pv_accumulator", "expect_overflow", "seed", "repetition", "cossim", "l1", "rmse",
    "overflow_events", "fp16_to_fp32_conversions", "mma_invocations", "wall_time",
]


def generate(shape, distribution: str = "gaussian", seed: int = 0, **params) -> np.ndarray:
    """Deterministic inputs with the reference generator's semantics (tensorio.py:41-88):
    Philox(seed); gaussian(mu, sigma) / uniform(low, high) / adversarial-max(magnitude); float32."""
    rng = np.random.Generator(np.random.Philox(seed))
    shape = tuple(int(s) for s in shape)
    if distribution == "gaussian":
        arr = rng.normal(float(params.pop("mu", 0.0)), float(params.pop("sigma", 1.0)), size=shape)
    elif distribution == "uniform":
        arr = rng.uniform(float(params.pop("low", 0.0)), float(params.pop("high", 1.0)), size=shape)
    elif distribution == "adversarial-max":
        arr = np.full(shape, float(params.pop("magnitude", 1.0)))
    else:
        raise ValueError(f"unknown distribution {distribution!r}")
    if params:
        raise ValueError(f"unused parameters for {distribution}: {sorted(params)}")
    return arr.astype(np.float32)


def exact_attention(q, k, v, causal: bool, scale: float, device: str = "cuda") -> np.ndarray:
    """FP64 softmax(Q K^T * scale) V on the GPU, per head (attention.py:186-220 semantics)."""
    tq, tk, tv = (torch.from_numpy(np.asarray(x, dtype=np.float64)).to(device) for x in (q, k, v))
    s = torch.einsum("hnd,hmd->hnm", tq, tk) * scale
    if causal:
        n = s.shape[-1]
        s = s.masked_fill(torch.triu(torch.ones(n, n, dtype=torch.bool, device=device), 1), float("-inf"))
    o = torch.softmax(s, dim=-1) @ tv
    return o.cpu().numpy()


def sweep(pairs, *, heads: int, seq_len: int, head_dim: int, seed: int = 0, repetitions: int = 1,
          distribution: str = "gaussian", causal: bool = False, smoothing: bool = True, qk_bits: int = 8,
          pv_accumulator: str = "fp16", params: dict | None = None, include_fp32_baseline: bool = False,
          inputs=None, out=sys.stderr) -> tuple[list[dict], bool]:
    """Rows for every valid pair (invalid ones are rejected loudly, as cli.py:253-259) and whether
    any unwaived pair overflowed the FP16 accumulator.  `inputs` = (q, k, v) overrides the generated
    ones (one repetition)."""
    triples = []
    for p_r, v_r, depth, *rest in pairs:
        waived = bool(rest[0]) if rest else False
        try:
            RangeConfig(p_r, v_r, depth, waived)
        except RangeConfigError as exc:
            print(f"rejected (p_r={p_r:g}, v_r={v_r:g}, depth={depth}): {exc}", file=out)
            continue
        triples.append((p_r, v_r, depth, waived, pv_accumulator))
    if include_fp32_baseline:
        triples.append((*FP32_BASELINE, True, "fp32"))
    rows, failed = [], False
    for rep in range(repetitions):
        s = seed + rep
        shape = (heads, seq_len, head_dim)
        if inputs is not None:
            q, k, v = inputs
        else:
            q = generate(shape, distribution, s, **dict(params or {}))
            k = generate(shape, distribution, s + 1, **dict(params or {}))
            v = generate(shape, distribution, s + 2, **dict(params or {}))
        reference = None
        for p_r, v_r, depth, waived, acc in triples:
            cfg = AttentionConfig(seq_len=seq_len, head_dim=head_dim, num_heads=heads, qk_bits=qk_bits,
                                  range=RangeConfig(p_r, v_r, depth, waived), causal=causal,
                                  smoothing=smoothing, pv_accumulator=acc)
            if reference is None:
                reference = exact_attention(q, k, v, causal, cfg.scale)
            t0 = time.perf_counter()
            report = attention_quantized(q, k, v, cfg)
            wall = time.perf_counter() - t0
            cos, l1, rmse = compare(reference, report.output)
            rows.append({
                "seq_len": seq_len, "head_dim": head_dim, "heads": heads, "block_q": cfg.block_q,
                "block_k": cfg.block_k, "qk_bits": qk_bits, "p_r": p_r, "v_r": v_r, "depth": depth,
                "causal": causal, "smoothing": smoothing, "pv_accumulator": acc, "expect_overflow": waived,
                "seed": s, "repetition": rep, "cossim": cos, "l1": l1, "rmse": rmse,
                "overflow_events": report.overflow_events,
                "fp16_to_fp32_conversions": report.fp16_to_fp32_conversions,
                "mma_invocations": report.mma_invocations, "wall_time": wall,
            })
            if report.overflow_events > 0 and not waived:
                print(f"error: unexpected overflow in (p_r={p_r:g}, v_r={v_r:g}, depth={depth})", file=out)
                failed = True
    return rows, failed


def to_csv(rows) -> str:
    buf = io.StringIO()
    w = csv.DictWriter(buf, fieldnames=REPORT_FIELDS, lineterminator="\n")
    w.writeheader()
    for r in rows:
        w.writerow(r)
    return buf.getvalue()


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2505_21136_b200.sweep")
    ap.add_argument("--preset", choices=["table2"], default=None)
    ap.add_argument("--spec", default=None, help="JSON with pairs / grid (cli.py:225-259 format)")
    ap.add_argument("--seq-len", type=int, default=256)
    ap.add_argument("--head-dim", type=int, default=64)
    ap.add_argument("--heads", type=int, default=1)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--repetitions", type=int, default=1)
    ap.add_argument("--causal", action="store_true")
    ap.add_argument("--no-smoothing", action="store_true")
    ap.add_argument("--qk-bits", type=int, default=8)
    ap.add_argument("--pv-accumulator", choices=["fp16", "fp32"], default="fp16")
    ap.add_argument("--fp32-baseline", action="store_true", help="add (448, 448, depth 1) with FP32 accumulation")
    ap.add_argument("--out", default=None)
    a = ap.parse_args(argv)
    pairs = [(p, v, d) for p, v, d in TABLE2_PAIRS] if a.preset == "table2" else []
    dist, params = "gaussian", {}
    if a.spec:
        spec = json.loads(Path(a.spec).read_text())
        for pr in spec.get("pairs", []):
            pairs.append((float(pr["p_r"]), float(pr["v_r"]), int(pr.get("depth", 2)),
                          bool(pr.get("expect_overflow", False))))
        grid = spec.get("grid")
        if grid:
            pairs += [(float(p), float(v), int(grid.get("depth", 2))) for p in grid["p_r"] for v in grid["v_r"]]
        inp = spec.get("input", {})
        dist, params = inp.get("distribution", "gaussian"), inp.get("parameters", {})
    if not pairs:
        print("sweep needs --preset and/or --spec with pairs or a grid", file=sys.stderr)
        return 2
    rows, failed = sweep(pairs, heads=a.heads, seq_len=a.seq_len, head_dim=a.head_dim, seed=a.seed,
                         repetitions=a.repetitions, distribution=dist, causal=a.causal,
                         smoothing=not a.no_smoothing, qk_bits=a.qk_bits, pv_accumulator=a.pv_accumulator,
                         params=params, include_fp32_baseline=a.fp32_baseline)
    text = to_csv(rows)
    if a.out:
        Path(a.out).write_text(text)
    else:
        sys.stdout.write(text)
    return 1 if failed else 0


if __name__ == "__main__":
    sys.exit(main())
