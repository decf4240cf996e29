"""The reference's own operator tests (lpattn tests/test_attention.py:173-265, class TestQuantized),
run through the B200 `attention_quantized` mirror with the same assertions.

The cases run at the reference's head_dim 32 (the 64-channel kernels on zero-padded channels) with
its seeds, shapes and thresholds unchanged.  Buffering depth 1 with the FP16 accumulator runs each
k=32 group as its own tcgen05 MMA into a fresh FP16 accumulator, converted and promoted on its own.
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

D = 32  # tests/test_attention.py uses head_dim 32


def gaussian_qkv(seed, heads, n, d):
    """tests/test_attention.py helper: Philox-seeded N(0,1) Q, K, V."""
    rng = np.random.Generator(np.random.Philox(seed))
    return tuple(rng.standard_normal((heads, n, d)) for _ in range(3))


def rel_err(a, b):
    return float(np.abs(a - b).sum() / np.abs(b).sum())


def exact(q, k, v, cfg):
    return oc.attention_reference(q, k, v, oc.AttentionConfig(
        seq_len=cfg.seq_len, head_dim=cfg.head_dim, num_heads=cfg.num_heads, causal=cfg.causal))


def test_all_zero_inputs():  # test_attention.py:174-179
    z = np.zeros((1, 64, D))
    rep = sa.attention_quantized(z, z, z, sa.AttentionConfig(seq_len=64, head_dim=D))
    assert not rep.output.any()
    assert rep.overflow_events == 0


def test_seq_len_one_recovers_value_row():  # test_attention.py:181-188
    q, k, v = gaussian_qkv(40, 1, 1, D)
    rep = sa.attention_quantized(q, k, v, sa.AttentionConfig(seq_len=1, head_dim=D))
    assert rel_err(rep.output, v) <= 2.0 ** -4
    assert rep.overflow_events == 0


def test_gaussian_close_to_reference():  # test_attention.py:190-198
    q, k, v = gaussian_qkv(41, 2, 256, D)
    cfg = sa.AttentionConfig(seq_len=256, head_dim=D, num_heads=2)
    rep = sa.attention_quantized(q, k, v, cfg)
    cos, _, _ = sa.compare(exact(q, k, v, cfg), rep.output)
    assert cos >= 0.999
    assert rep.overflow_events == 0
    # the reference's bound is 1/p_r + 1e-12 in FP64; the kernel's delta_P is an f32 (1 ulp = 2^-23 rel.)
    assert rep.p_scale_max <= (1.0 / cfg.range.p_r) * (1 + 2.0 ** -23)


@pytest.mark.parametrize("causal", [False, True])
def test_ragged_seq_len_padding(causal):  # test_attention.py:200-208 (block_q 128 here)
    q, k, v = gaussian_qkv(42, 1, 100, D)
    cfg = sa.AttentionConfig(seq_len=100, head_dim=D, causal=causal)
    rep = sa.attention_quantized(q, k, v, cfg)
    cos, _, _ = sa.compare(exact(q, k, v, cfg), rep.output)
    assert cos >= 0.995


def test_int4_mode():  # test_attention.py:210-215
    q, k, v = gaussian_qkv(43, 1, 128, D)
    cfg = sa.AttentionConfig(seq_len=128, head_dim=D, qk_bits=4)
    rep = sa.attention_quantized(q, k, v, cfg)
    cos, _, _ = sa.compare(exact(q, k, v, cfg), rep.output)
    assert cos >= 0.95


def test_conversion_halving_at_run_level():  # test_attention.py:217-230
    q, k, v = gaussian_qkv(44, 1, 128, D)
    reports = {}
    for depth in (1, 2):
        config = sa.AttentionConfig(seq_len=128, head_dim=D, range=sa.RangeConfig(224.0, 4.5, depth))
        reports[depth] = sa.attention_quantized(q, k, v, config)
    assert reports[1].fp16_to_fp32_conversions == 2 * reports[2].fp16_to_fp32_conversions
    assert reports[1].mma_invocations == reports[2].mma_invocations
    # the depth-1 run is a real FP16-per-group computation on the GPU: close to depth 2 and to the oracle
    cfg = oc.AttentionConfig(seq_len=128, head_dim=D, range=oc.RangeConfig(224.0, 4.5, 1))
    want = oc.attention_quantized(q, k, v, cfg).output
    assert sa.compare(want, reports[1].output)[0] >= 0.9999
    assert sa.compare(reports[2].output, reports[1].output)[0] >= 0.9999


def test_fp32_baseline_close_to_fp16_path():  # test_attention.py:232-245
    q, k, v = gaussian_qkv(45, 1, 128, D)
    fast = sa.attention_quantized(q, k, v, sa.AttentionConfig(seq_len=128, head_dim=D))
    baseline = sa.attention_quantized(q, k, v, sa.AttentionConfig(
        seq_len=128, head_dim=D, pv_accumulator="fp32",
        range=sa.RangeConfig(448.0, 448.0, 1, expect_overflow=True)))
    ref = exact(q, k, v, sa.AttentionConfig(seq_len=128, head_dim=D))
    assert baseline.overflow_events == 0
    assert baseline.fp16_to_fp32_conversions == 0
    c_fast, _, _ = sa.compare(ref, fast.output)
    c_base, _, _ = sa.compare(ref, baseline.output)
    assert abs(c_fast - c_base) <= 1e-3


def test_unsafe_ranges_overflow_on_adversarial_input():  # test_attention.py:247-254
    """(448, 448) at depth 2 on all-ones inputs: every P^ and V^ code is 448, 64 products of 448^2
    overflow the FP16 accumulator of the real tensor core (inf, counted at promotion)."""
    ones = np.full((1, 64, D), 1.0)
    cfg = sa.AttentionConfig(seq_len=64, head_dim=D,
                             range=sa.RangeConfig(448.0, 448.0, 2, expect_overflow=True))
    rep = sa.attention_quantized(ones, ones, ones, cfg)
    assert rep.overflow_events > 0


def test_safe_ranges_do_not_overflow_on_adversarial_input():
    """The paper's (224, 4.5) pair on the same adversarial input stays finite (Table 2)."""
    ones = np.full((1, 64, D), 1.0)
    rep = sa.attention_quantized(ones, ones, ones, sa.AttentionConfig(seq_len=64, head_dim=D))
    assert rep.overflow_events == 0
    assert np.allclose(rep.output, 1.0, rtol=2.0 ** -4)


def test_smoothing_helps_with_a_common_mode():  # test_attention.py:255-261
    q, k, v = gaussian_qkv(46, 1, 128, D)
    q = q + 4.0  # large common mode that smoothing removes
    ref = exact(q, k, v, sa.AttentionConfig(seq_len=128, head_dim=D))
    on = sa.attention_quantized(q, k, v, sa.AttentionConfig(seq_len=128, head_dim=D, smoothing=True))
    off = sa.attention_quantized(q, k, v, sa.AttentionConfig(seq_len=128, head_dim=D, smoothing=False))
    assert sa.compare(ref, on.output)[0] >= sa.compare(ref, off.output)[0]


def test_head_dim_must_be_multiple_of_32():  # test_attention.py:263-266
    q, k, v = gaussian_qkv(47, 1, 64, 16)
    with pytest.raises(ValueError):
        sa.attention_quantized(q, k, v, sa.AttentionConfig(seq_len=64, head_dim=16))


def test_block_k_must_be_multiple_of_32():  # test_attention.py:268-273
    q, k, v = gaussian_qkv(48, 1, 64, D)
    with pytest.raises(ValueError):
        sa.attention_quantized(q, k, v, sa.AttentionConfig(seq_len=64, head_dim=D, block_k=48))


def test_causal_quantized_matches_reference():  # test_attention.py:275-281
    q, k, v = gaussian_qkv(49, 1, 256, D)
    cfg = sa.AttentionConfig(seq_len=256, head_dim=D, causal=True)
    rep = sa.attention_quantized(q, k, v, cfg)
    cos, _, _ = sa.compare(exact(q, k, v, cfg), rep.output)
    assert cos >= 0.999
    assert rep.overflow_events == 0


def test_lpattn_tensor_fixture_through_the_gpu():
    """CPU <-> GPU exchange in the reference's LPATTN-TENSOR v1 files: Q/K/V
    written by the unmodified reference's `gen` path are loaded straight onto the device with
    tensorio.load, run through the attention_quantized mirror, and checked against the reference's
    output file and run row (tests/golden/make_tensor_fixtures.py)."""
    import json
    from pathlib import Path

    from paper_2505_21136_b200 import tensorio

    fix = Path(__file__).resolve().parent / "golden" / "lpattn_tensor"
    row = json.loads((fix / "run.json").read_text())
    q, k, v = (tensorio.load(fix / f"{n}.bin", device="cuda") for n in ("q", "k", "v"))
    assert q.is_cuda and q.shape == (row["heads"], row["seq_len"], row["head_dim"])
    cfg = sa.AttentionConfig(seq_len=row["seq_len"], head_dim=row["head_dim"], num_heads=row["heads"])
    rep = sa.attention_quantized(q.cpu().numpy(), k.cpu().numpy(), v.cpu().numpy(), cfg)
    ref_out = tensorio.read_tensor(fix / "out.bin").astype(np.float64)
    cos, l1, _ = sa.compare(ref_out, rep.output)
    assert cos >= 0.9999 and l1 <= 1e-3, (cos, l1)
    assert rep.overflow_events == row["overflow_events"]
    assert rep.fp16_to_fp32_conversions == row["fp16_to_fp32_conversions"]
    assert rep.mma_invocations == row["mma_invocations"]
    ex = exact(q.cpu().double().numpy(), k.cpu().double().numpy(), v.cpu().double().numpy(), cfg)
    cos_x, l1_x, _ = sa.compare(ex, rep.output)
    assert cos_x >= row["cossim"] - 1e-4 and l1_x <= row["l1"] + 1e-3, (cos_x, l1_x, row)
    out_path = Path("/tmp") / "sa2pp_fixture_out.bin"
    tensorio.save(out_path, torch.from_numpy(rep.output))  # and back into the reference's format
    assert np.allclose(tensorio.read_tensor(out_path), rep.output.astype(np.float32))
