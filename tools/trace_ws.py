"""Per-phase clock trace of the warp-specialised attention kernel (development aid; needs a GPU).

Every tile of heads 0-2 is traced (INSTR build: clock64 per block < 64, warp, phase).  CTAs that ran
on the same SM at the same time are paired, and their per-block phase times are printed on the
SM's clock, relative to the first CTA's softmax warp 0 entering block j.
Softmax warps 0-3: 0 enter, 1 S ready, 2 published max-shift (waiting for the tile max),
3 tile max known, 4 P^ stored.  Promotion warps 4-7: 0 enter, 1 stage visible, 2 PV ready,
3 promoted; warp 4 also 8 p_ready seen, 9 pv_free seen, 12 PV/S(j+2)/refill issued.
    python tools/trace_ws.py [N] [fp16|fp32] [D] [causal]
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2505_21136_b200 as sa
from paper_2505_21136_b200 import _abi as A

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
acc = sys.argv[2] if len(sys.argv) > 2 else "fp16"
D = int(sys.argv[3]) if len(sys.argv) > 3 else 128
causal = len(sys.argv) > 4 and sys.argv[4] == "causal"
q = torch.randn(4, 32, N, D, device="cuda", dtype=torch.bfloat16)
k, v = torch.randn_like(q), torch.randn_like(q)
sa.sageattn(q, k, v, is_causal=causal, pv_accum=acc)
n_qt = (N + 127) // 128
tr = torch.zeros(3 * n_qt * 66 * 128, dtype=torch.int64, device="cuda")
A.lib().sa2pp_set_trace_buffer(tr.data_ptr())
sa.sageattn(q, k, v, is_causal=causal, pv_accum=acc)
torch.cuda.synchronize()
A.lib().sa2pp_set_trace_buffer(None)
t = tr.view(3 * n_qt, 66, 128).cpu().numpy().astype(np.int64)
ctas = [c for c in range(3 * n_qt) if t[c, 0, 3] > 0]
# pair CTAs on the same SM whose block-0 entry clocks are within one block period
by_sm = {}
for c in ctas:
    by_sm.setdefault(int(t[c, 0, 0]), []).append(c)
pairs = []
for sm, cs in by_sm.items():
    cs.sort(key=lambda c: t[c, 2, 0])
    for a_, b_ in zip(cs, cs[1:]):
        if abs(t[a_, 2 + 8, 0] - t[b_, 2 + 8, 0]) < 200000:
            pairs.append((sm, a_, b_))
print(f"traced CTAs {len(ctas)}, co-resident pairs {len(pairs)}")
names = {0: "enter", 1: "S", 2: "pub", 3: "tmax", 4: "P^", 8: "prdy", 9: "pvfree", 12: "issued"}
for sm, ca, cb in pairs[:3]:
    print(f"--- SM {sm}: CTA {ca} and CTA {cb}")
    for j in range(8, 16):
        base = t[ca, 2 + j, 0]
        for c in (ca, cb):
            row = t[c, 2 + j]
            sm_ = " ".join(f"{names[k]}:{row[k] - base:+6d}" for k in (0, 1, 2, 3, 4))
            pr = " ".join(f"{k}:{row[16 * 4 + k] - base:+6d}" for k in (0, 1, 2, 3, 8, 9, 12))
            print(f"  j={j} cta{c % 1000:4d} softmax w0 [{sm_}]  promo w4 [{pr}]")
for c in ctas[:1]:
    blk = t[c, 2:2 + 64]
    per = np.median(np.diff(blk[4:60, 0]))
    print(f"median block period of CTA {c}: {per:.0f} clk")
