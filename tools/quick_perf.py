"""Quick device timing of prepass and attention kernels (development aid, not the bench)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2505_21136_b200 as sa
from paper_2505_21136_b200 import api, _abi as A
import ctypes


def time_ms(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    B, H, D = 4, 32, 128
    for N in [int(x) for x in (sys.argv[1:] or ["1024", "4096", "16384"])]:
        for causal in (False, True):
            for acc in ("fp16", "fp32"):
                q = torch.randn(B, H, N, D, device="cuda", dtype=torch.bfloat16)
                k = torch.randn_like(q)
                v = torch.randn_like(q)
                out, qt = sa.sageattn(q, k, v, is_causal=causal, pv_accum=acc, return_quant=True)
                prob = api._problem(B, H, H, N, D, causal=causal, pv_accum=acc)
                o = A.Output(A.SA2PP_BF16, out.data_ptr(), (ctypes.c_int64 * 3)(*[out.stride(i) for i in range(3)]))
                qs = qt.struct()
                stream = torch.cuda.current_stream().cuda_stream
                attn = lambda: A.check(A.lib().sa2pp_attn_fwd(ctypes.byref(prob), ctypes.byref(qs), ctypes.byref(o), None, stream))
                full = lambda: sa.sageattn(q, k, v, is_causal=causal, pv_accum=acc, out=out, quant=qt)
                ta = time_ms(attn)
                tf = time_ms(full)
                ops = 4 * B * H * N * N * D * (0.5 if causal else 1.0)
                print(f"N={N:6d} causal={int(causal)} acc={acc}: attn {ta:8.3f} ms {ops/ta/1e9:8.1f} TOPS | "
                      f"sageattn {tf:8.3f} ms {ops/tf/1e9:8.1f} TOPS", flush=True)


if __name__ == "__main__":
    main()
