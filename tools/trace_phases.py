"""Per-phase clock trace of a few attention CTAs (development aid; needs a GPU).

Stamps per block and warp (lane 0): 0 S ready, 1 S loaded, 2 pass 1 done, 3 after the pair
barrier, 4 after the tile-max wait, 5 pass 2 packed, 6 PV(j-1) ready (in the promotion),
7 block end; MMA issuer only: 8 enter, 9 blk_done(j-1) seen,
10 PV(j-1) issued, 11 S(j+1) issued; 13 published (h=0), 14 before the tile-max wait.
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
q = torch.randn(4, 32, N, D, device="cuda", dtype=torch.bfloat16)
k, v = torch.randn_like(q), torch.randn_like(q)
sa.sageattn(q, k, v, pv_accum=acc)
tr = torch.zeros(8 * 66 * 128, dtype=torch.int64, device="cuda")
A.lib().sa2pp_set_trace_buffer(tr.data_ptr())
sa.sageattn(q, k, v, pv_accum=acc)
torch.cuda.synchronize()
A.lib().sa2pp_set_trace_buffer(None)
t = tr.view(8, 66, 128).cpu().numpy().astype(np.int64)
names = ["S-ready", "ldS", "pass1", "pairbar", "dt-wait", "pass2", "PV-ready", "end"]
for cta in range(2):
    smid, g0, g1, nb = t[cta, 0, :4]
    nb = min(int(nb), 64)
    blk = t[cta, 2:2 + nb, :]
    base = blk[:, 0]  # warp 0 S-ready
    print(f"cta{cta} sm{smid} blocks {nb} duration {(g1 - g0) / 1e3:.1f} us")
    for w in range(8):
        ph = blk[:, 16 * w:16 * w + 8]
        sl = slice(4, nb - 2)
        rel = [np.median(ph[sl, k] - base[sl]) for k in range(8)]
        per = np.median(np.diff(ph[2:nb, 0]))
        x13 = np.median(blk[sl, 16 * w + 13] - base[sl]) if blk[5, 16 * w + 13] else float("nan")
        x14 = np.median(blk[sl, 16 * w + 14] - base[sl])
        print(f"  warp{w} block {per:6.0f} | " + " ".join(f"{names[k]} {rel[k]:+6.0f}" for k in range(8))
              + f" | published {x13:+6.0f} pre-dt-wait {x14:+6.0f}")
    iss = []
    for w in range(8):
        for j in range(4, nb - 2):
            s_ = blk[j, 16 * w + 8:16 * w + 12]
            if s_[0] > 0:
                iss.append((w, s_ - s_[0], s_[0] - base[j]))
    if iss:
        ws = [w for w, _, _ in iss]
        arr = np.array([x for _, x, _ in iss])
        at = np.array([a for _, _, a in iss])
        print(f"  MMA issuer warps {np.bincount(ws, minlength=8).tolist()}; enter at {np.median(at):+.0f}; "
              f"blk_done +{np.median(arr[:, 1]):.0f}, PV(j-1) issued +{np.median(arr[:, 2]):.0f}, "
              f"S(j+1) issued +{np.median(arr[:, 3]):.0f}")
