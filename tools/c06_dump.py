"""Dump the B200 outputs for the reference's acceptance test c06 inputs (tests/test_acceptance.py:
187-220: 8x1024x128, one Philox(0) stream for q, k, v) so they can be compared with the reference's
outputs on the CPU.  Development aid."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2505_21136_b200 import AttentionConfig, RangeConfig, attention_quantized  # noqa: E402

out = Path(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c06")
out.mkdir(parents=True, exist_ok=True)
heads, seq, dim = 8, 1024, 128
rng = np.random.Generator(np.random.Philox(0))
q, k, v = (rng.normal(size=(heads, seq, dim)) for _ in range(3))
base = AttentionConfig(seq_len=seq, head_dim=dim, num_heads=heads)
for p_r, v_r in [(448.0, 2.25), (224.0, 4.5), (112.0, 9.0)]:
    r = attention_quantized(q, k, v, base.with_range(RangeConfig(p_r, v_r, 2)))
    np.save(out / f"ours_{p_r}_{v_r}.npy", r.output.astype(np.float32))
cfg = AttentionConfig(seq_len=seq, head_dim=dim, num_heads=heads, pv_accumulator="fp32",
                      range=RangeConfig(448.0, 448.0, 1, expect_overflow=True))
r = attention_quantized(q, k, v, cfg)
np.save(out / "ours_fp32.npy", r.output.astype(np.float32))
cfg16 = AttentionConfig(seq_len=seq, head_dim=dim, num_heads=heads, pv_accumulator="fp16",
                        range=RangeConfig(448.0, 448.0, 1, expect_overflow=True))
print("done")
