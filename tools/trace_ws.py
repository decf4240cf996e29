"""Per-phase clock trace of the warp-specialised attention kernel (development aid; needs a GPU).

Softmax warps 0-3: 0 enter, 1 S ready, 2 published max-shift, 3 tile max known, 4 P^ ready.
Promotion warps 4-7: 0 enter (warp 4 issues PV(j)/S(j+2) next), 1 stage visible, 2 PV ready, 3 promoted;
warp 4 also 8 p_ready seen, 9 pv_free seen, 10 PV issued, 11 K(j+2) landed, 12 S(j+2)+refill issued.
    python tools/trace_ws.py [N] [fp16|fp32] [D] [causal]
"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2505_21136_b200 as sa
from paper_2505_21136_b200 import _abi as A

N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
acc = sys.argv[2] if len(sys.argv) > 2 else "fp16"
D = int(sys.argv[3]) if len(sys.argv) > 3 else 128
causal = len(sys.argv) > 4 and sys.argv[4] == "causal"
q = torch.randn(4, 32, N, D, device="cuda", dtype=torch.bfloat16)
k, v = torch.randn_like(q), torch.randn_like(q)
sa.sageattn(q, k, v, is_causal=causal, pv_accum=acc)
tr = torch.zeros(8 * 66 * 128, dtype=torch.int64, device="cuda")
A.lib().sa2pp_set_trace_buffer(tr.data_ptr())
sa.sageattn(q, k, v, is_causal=causal, pv_accum=acc)
torch.cuda.synchronize()
A.lib().sa2pp_set_trace_buffer(None)
t = tr.view(8, 66, 128).cpu().numpy().astype(np.int64)
for cta in range(3):
    smid, g0, g1, nb = t[cta, 0, :4]
    nb = min(int(nb), 64)
    blk = t[cta, 2:2 + nb, :]
    base = blk[:, 16 * 4]  # warp 4 (promotion) enters iteration j
    sl = slice(6, nb - 2)
    per = np.median(np.diff(blk[4:nb, 16 * 4]))
    print(f"cta{cta} sm{smid} blocks {nb} duration {(g1 - g0) / 1e3:.1f} us; block period {per:.0f} clk "
          "(times relative to warp 4 entering iteration j)")
    for w in range(8):
        ks = [k for k in range(16) if blk[sl, 16 * w + k].max() > 0]
        rel = {}
        for k in ks:
            m = blk[sl, 16 * w + k] > 0
            rel[k] = np.median(blk[sl, 16 * w + k][m] - base[sl][m])
        print(f"  warp{w}: " + " ".join(f"{k}:{rel[k]:+6.0f}" for k in ks))
