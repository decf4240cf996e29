import torch, sys
sys.path.insert(0, '.')
import paper_2505_21136_b200 as sa
from paper_2505_21136_b200 import api, _abi as A
import ctypes
def run(B, H, N, D=128, causal=False, iters=20):
    q = torch.randn(B, H, N, D, device='cuda').bfloat16(); k = torch.randn_like(q); v = torch.randn_like(q)
    out, qt = sa.sageattn(q, k, v, is_causal=causal, return_quant=True)
    prob = api._problem(B, H, H, N, D, causal=causal)
    o = A.Output(A.SA2PP_BF16, out.data_ptr(), (ctypes.c_int64 * 3)(out.stride(0), out.stride(1), out.stride(2)))
    qs = qt.struct(); lib = A.lib(); s = torch.cuda.current_stream().cuda_stream
    for _ in range(3): lib.sa2pp_attn_fwd(ctypes.byref(prob), ctypes.byref(qs), ctypes.byref(o), None, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): lib.sa2pp_attn_fwd(ctypes.byref(prob), ctypes.byref(qs), ctypes.byref(o), None, s)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    ops = 4 * B * H * N * N * D * (0.5 if causal else 1)
    ctas = B * H * ((N + 127) // 128)
    print(f"B={B} H={H} N={N} causal={causal} ctas={ctas} waves={ctas/296:.2f} {ms*1e3:.1f} us {ops/ms/1e9:.1f} TOPS", flush=True)
for (B, H, N) in [(4, 32, 1024), (37, 32, 1024), (4, 32, 2048), (37, 16, 2048), (4, 32, 4096), (37, 8, 4096)]:
    run(B, H, N)
for (B, H, N) in [(4, 32, 1024), (37, 32, 1024), (4, 32, 2048), (37, 16, 2048)]:
    run(B, H, N, causal=True)
