"""Range sweep harness (paper_2505_21136_b200/sweep.py), SURVEY §8(f1)."""

import numpy as np
import pytest

from conftest import gpu_ready


def test_generator_matches_reference(lpattn):
    from lpattn import tensorio
    from paper_2505_21136_b200.sweep import generate
    for dist, params in (("gaussian", {}), ("gaussian", {"mu": 1.0, "sigma": 2.0}), ("uniform", {}),
                         ("adversarial-max", {"magnitude": 3.0})):
        ref, _ = tensorio.generate((2, 33, 16), dist, 7, **dict(params))
        assert np.array_equal(generate((2, 33, 16), dist, 7, **dict(params)), ref)


def test_report_fields_match_reference(lpattn):
    from lpattn import cli
    from paper_2505_21136_b200.sweep import REPORT_FIELDS, TABLE2_PAIRS
    assert REPORT_FIELDS == cli.REPORT_FIELDS
    assert TABLE2_PAIRS == cli.TABLE2_PAIRS


@pytest.mark.gpu
def test_table2_acceptance_c06_on_b200():
    """tests/test_acceptance.py:187-220 of the reference, on the sm_100a path and on its inputs
    (8x1024x128, one Philox(0) stream for q, k, v): every Table-2 pair and the FP32 SageAttention2
    baseline within 1e-3 cossim / 2e-4 L1 of each other, each >= 0.999 cossim against exact
    attention, no unwaived overflow.  (The L1 spread bound is a property of these inputs: on the
    CLI's seed-per-tensor inputs the reference itself spreads 4.7e-4, and so does this path.)"""
    if not gpu_ready():
        pytest.skip("needs a CUDA device")
    from paper_2505_21136_b200.sweep import TABLE2_PAIRS, sweep
    rng = np.random.Generator(np.random.Philox(0))
    qkv = tuple(rng.normal(size=(8, 1024, 128)) for _ in range(3))
    rows, failed = sweep(TABLE2_PAIRS, heads=8, seq_len=1024, head_dim=128, seed=0,
                         include_fp32_baseline=True, inputs=qkv)
    assert not failed
    assert len(rows) == 4
    cos = [r["cossim"] for r in rows]
    l1 = [r["l1"] for r in rows]
    assert min(cos) >= 0.999, cos
    assert max(cos) - min(cos) <= 1e-3, cos
    assert max(l1) - min(l1) <= 2e-4, l1
    assert all(r["overflow_events"] == 0 for r in rows[:3])
    # the reference's own numbers on these inputs (lpattn 8x1024x128, measured in the build container)
    ref_l1 = [0.03683061507916469, 0.03683199871979319, 0.036832208253615814, 0.036833232136791974]
    assert all(abs(a - b) <= 2e-5 for a, b in zip(l1, ref_l1)), (l1, ref_l1)
