"""PCIe probe for the end-to-end path: H2D / D2H / bidirectional bandwidth of pinned buffers, and
HostPipeline step time at the bench shape for several chunkings.  python tools/pcie_probe.py"""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2505_21136_b200 as sa  # noqa: E402

dev = torch.device("cuda:0")
GB = 1e9


def timeit(fn, n=3):
    fn()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(n):
        fn()
    s1.record()
    torch.cuda.synchronize()
    return s0.elapsed_time(s1) / n


nb = 1610612736
h_in = torch.empty(nb, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(nb, dtype=torch.uint8, device=dev)
nbo = 536870912
h_out = torch.empty(nbo, dtype=torch.uint8, pin_memory=True)
d_out = torch.empty(nbo, dtype=torch.uint8, device=dev)
ms = timeit(lambda: d_in.copy_(h_in, non_blocking=True))
print(f"H2D {nb/GB:.2f} GB: {ms:.2f} ms = {nb/ms/1e6:.1f} GB/s")
ms = timeit(lambda: h_out.copy_(d_out, non_blocking=True))
print(f"D2H {nbo/GB:.2f} GB: {ms:.2f} ms = {nbo/ms/1e6:.1f} GB/s")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        for _ in range(3):
            h_out.copy_(d_out, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


ms = timeit(both)
print(f"bidirectional H2D {nb/GB:.2f} GB + D2H {3*nbo/GB:.2f} GB: {ms:.2f} ms")
# chunked H2D (16 pieces) back to back
ch = nb // 16
ms = timeit(lambda: [d_in[i * ch:(i + 1) * ch].copy_(h_in[i * ch:(i + 1) * ch], non_blocking=True) for i in range(16)])
print(f"H2D 16 chunks: {ms:.2f} ms = {nb/ms/1e6:.1f} GB/s")
del h_in, d_in, h_out, d_out

B, H, N, D = 4, 32, 16384, 128
q, k, v = (torch.randn(B, H, N, D, dtype=torch.bfloat16) .pin_memory() for _ in range(3))
o = torch.empty_like(q).pin_memory()
ops = 4 * B * H * N * N * D
for chunks, depth in ((16, 3), (32, 3), (32, 4), (64, 3), (64, 4)):
    pipe = sa.HostPipeline(1, B * H, B * H, N, D, torch.bfloat16, dev, chunks=chunks, depth=depth)
    qf, kf, vf, of = (t.view(1, B * H, N, D) for t in (q, k, v, o))
    ms = timeit(lambda: pipe(qf, kf, vf, of), n=5)
    print(f"HostPipeline chunks={chunks} depth={depth}: {ms:.2f} ms/step = {ops/ms/1e9:.1f} TOPS")
    del pipe
