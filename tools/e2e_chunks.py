"""e2e (pinned host arrays through HostPipeline) ms per call vs chunk count and ring depth.

    python tools/e2e_chunks.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2505_21136_b200 as sa  # noqa: E402

SHAPES = {"kernel": (4, 32, 16384, 128, False), "causal": (4, 32, 16384, 128, True),
          "cogvideox": (2, 30, 17776, 64, False)}
dev = torch.device("cuda:0")
for name, (B, H, N, D, causal) in SHAPES.items():
    g = torch.Generator().manual_seed(0)
    hq, hk, hv = (torch.randn(B, H, N, D, generator=g).bfloat16().pin_memory() for _ in range(3))
    ho = torch.empty_like(hq).pin_memory()
    for chunks in (8, 16, 32, 64):
        for depth in (2, 3, 4):
            pipe = sa.HostPipeline(B, H, H, N, D, torch.bfloat16, dev, is_causal=causal, chunks=chunks, depth=depth)
            for _ in range(2):
                pipe(hq, hk, hv, ho)
            torch.cuda.synchronize()
            s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            for _ in range(4):
                pipe(hq, hk, hv, ho)
            s1.record()
            torch.cuda.synchronize()
            print(f"{name} chunks={chunks} depth={depth} ms={s0.elapsed_time(s1) / 4:.2f}", flush=True)
            del pipe
