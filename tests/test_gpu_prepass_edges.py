"""Prepass bit-exactness on adversarial inputs (GPU vs the CPU oracle).

The sm_100a prepass computes Q/K INT8 codes and V E4M3 codes with an FP32 fast path and falls back to
the FP64 quotient near rounding ties, and when |mean| is large against the tile's amplitude
(csrc/prepass.cu: int_code_fast, e4m3_div_fast).  These cases put values exactly on and next to the
ties, use huge channel offsets, zeros and subnormals, and check every code against the oracle's
restatement of the reference (quantization.py:151-160, 178-188; numerics.py:152-182).
"""

import numpy as np
import pytest

from conftest import gpu_ready

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not gpu_ready():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2505_21136_b200 as sa  # noqa: E402
from oracle import sage_cpu as oc  # noqa: E402
from edge_inputs import CASES  # noqa: E402


def _check(q, k, v, smoothing=True):
    h, n, d = q.shape
    cfg = oc.AttentionConfig(seq_len=n, head_dim=d, num_heads=h, smoothing=smoothing)
    qt = sa.quantize(*(torch.from_numpy(x[None]).cuda() for x in (q, k, v)), smooth=smoothing)
    torch.cuda.synchronize()
    for hh in range(h):
        ref = oc.prepass(q[hh], k[hh], v[hh], cfg)
        assert np.array_equal(qt.q_codes[0, hh].cpu().numpy()[:n], ref.q_codes), f"Q codes head {hh}"
        assert np.array_equal(qt.q_scale64[0, hh].cpu().numpy(), ref.q_scale), f"Q scales head {hh}"
        assert np.array_equal(qt.k_codes[0, hh].cpu().numpy(), ref.k_codes), f"K codes head {hh}"
        assert np.array_equal(qt.k_scale64[0, hh].cpu().numpy(), ref.k_scale), f"K scales head {hh}"
        assert np.array_equal(qt.v_codes[0, hh].cpu().numpy().T, ref.v_codes), f"V codes head {hh}"
        assert np.array_equal(qt.v_scale64[0, hh].cpu().numpy(), ref.v_scale), f"V scales head {hh}"


@pytest.mark.parametrize("case", sorted(CASES))
def test_prepass_edges_bit_exact(case):
    q, k, v, smoothing = CASES[case]()
    _check(q, k, v, smoothing=smoothing)
