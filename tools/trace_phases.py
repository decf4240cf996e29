"""Per-phase clock trace of a few attention CTAs (development aid; needs a GPU).

Stamps per block (thread 0 and thread 128): 0 S ready, 1 S loaded, 2 pass-1 done, 3 after the
tile-max barrier, 4 t reloaded, 5 exp/pack done, 6 PV(j-1) ready, 7 promotion done.
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
q = torch.randn(4, 32, N, 128, device="cuda", dtype=torch.bfloat16)
k, v = torch.randn_like(q), torch.randn_like(q)
sa.sageattn(q, k, v, pv_accum=acc)
tr = torch.zeros(8 * 66 * 64, dtype=torch.int64, device="cuda")
A.lib().sa2pp_set_trace_buffer(tr.data_ptr())
sa.sageattn(q, k, v, pv_accum=acc)
torch.cuda.synchronize()
A.lib().sa2pp_set_trace_buffer(None)
t = tr.view(8, 66, 64).cpu().numpy().astype(np.int64)
names = ["S-wait", "ldS", "pass1", "barrier", "ldT", "exp", "PVwait", "promote", "end->next"]
for cta in range(2):
    smid, g0, g1, nb = t[cta, 0, :4]
    base = t[cta, 2:2 + min(int(nb), 64), 0].copy()
    for w in range(8):
        th = 8 * w
        ph = t[cta, 2:2 + min(int(nb), 64), th:th + 8]
        arr2 = np.median(ph[2:-1, 2] - base[2:-1])
        print(f"  warp{w}: pass1-done at +{arr2:.0f} vs warp0 block start, S-ready at +{np.median(ph[2:-1,0]-base[2:-1]):.0f}")
        nbl = ph.shape[0]
        d = [np.median(ph[2:nbl - 1, k + 1] - ph[2:nbl - 1, k]) for k in range(7)]
        nxt = np.median(ph[3:nbl, 0] - ph[2:nbl - 1, 7])
        blk = np.median(np.diff(ph[2:nbl, 0]))
        print(f"cta{cta} sm{smid} warp{w} blk {blk:5.0f} | " + " ".join(
            f"{names[k + 1]} {d[k]:5.0f}" for k in range(7)) + f" | {names[8]} {nxt:5.0f}")
