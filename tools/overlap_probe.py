"""Does running the prepass of chunk i+1 beside the attention kernel of chunk i hide the prepass?
Chunks are batches of the headline shape; two quant buffer sets ping-pong.  python tools/overlap_probe.py"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2505_21136_b200 as sa  # noqa: E402
from paper_2505_21136_b200 import _abi as A  # noqa: E402
from paper_2505_21136_b200.api import C_ref, _problem, alloc_quant  # noqa: E402

dev = torch.device("cuda:0")
B, H, N, D = 4, 32, 16384, 128
q, k, v = (torch.randn(B, H, N, D, device=dev, dtype=torch.bfloat16) for _ in range(3))
out = torch.empty_like(q)
ops = 4 * B * H * N * N * D


def run(nch, overlap, prio=None):
    bc = B // nch
    prob = _problem(bc, H, H, N, D, causal=False)
    sets = [alloc_quant(prob, dev) for _ in range(2)]
    lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
    sp = torch.cuda.Stream(priority=(hi if prio == "pre_hi" else 0))
    sa_ = torch.cuda.Stream(priority=(hi if prio == "attn_hi" else 0))
    evp = [torch.cuda.Event() for _ in range(nch)]
    eva = [torch.cuda.Event() for _ in range(nch)]
    lib = A.lib()

    def step():
        cur = torch.cuda.current_stream()
        sp.wait_stream(cur)
        sa_.wait_stream(cur)
        for i in range(nch):
            qt = sets[i % 2]
            st = sp if overlap else sa_
            if overlap and i >= 2:
                sp.wait_event(eva[i - 2])
            sl = slice(i * bc, (i + 1) * bc)
            qi, ki, vi, oi = q[sl], k[sl], v[sl], out[sl]
            strides = lambda t: (A.C.c_int64 * 3)(*t.stride()[:3])  # noqa: E731
            ins = A.Inputs(A.SA2PP_BF16, qi.data_ptr(), ki.data_ptr(), vi.data_ptr(), strides(qi), strides(ki),
                           strides(vi))
            A.check(lib.sa2pp_prepass(C_ref(prob), C_ref(ins), C_ref(qt.struct()), qt.workspace.data_ptr(),
                                      qt.workspace.numel(), st.cuda_stream))
            evp[i].record(st)
            sa_.wait_event(evp[i])
            o = A.Output(A.SA2PP_BF16, oi.data_ptr(), strides(oi))
            A.check(lib.sa2pp_attn_fwd(C_ref(prob), C_ref(qt.struct()), C_ref(o), None, sa_.cuda_stream))
            eva[i].record(sa_)
        cur.wait_stream(sa_)
        cur.wait_stream(sp)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"chunks={nch} overlap={overlap} prio={prio}: {ms:.3f} ms = {ops / ms / 1e9:.1f} TOPS", flush=True)
    ref = sa.sageattn(q, k, v)
    assert torch.equal(ref, out)


run(1, False)
for nch in (2, 4):
    run(nch, False)
    run(nch, True)
    run(nch, True, "pre_hi")
    run(nch, True, "attn_hi")
