"""Pin the numpy restatement (oracle/sage_cpu.py) to the reference's own numbers.

CPU only.  The fixtures were produced by the unmodified reference
(tests/golden/make_golden.py); where the reference source tree exists, a few
extra checks also run it live on fresh seeds.
"""

import math

import numpy as np
import pytest

from conftest import golden_cases, load_golden
from oracle import sage_cpu as oc


def cfg_from(g) -> oc.AttentionConfig:
    seq, dim, heads, causal, smoothing, qk_bits, fp16, depth, waive = (int(x) for x in g["cfg"])
    p_r, v_r, sm = (float(x) for x in g["ranges"])
    return oc.AttentionConfig(
        seq_len=seq, head_dim=dim, num_heads=heads, causal=bool(causal), smoothing=bool(smoothing),
        qk_bits=qk_bits, pv_accumulator="fp16" if fp16 else "fp32",
        range=oc.RangeConfig(p_r, v_r, depth, bool(waive)),
        softmax_scale=None if sm < 0 else sm)


# ------------------------------------------------------------------ codecs (numerics.py)
class TestCodec:
    def test_decode_table_matches_reference(self):
        g = load_golden("codec")
        got = oc.e4m3_decode(np.arange(256))
        same = (got == g["decoded"]) | (np.isnan(got) & np.isnan(g["decoded"]))
        assert same.all()

    def test_encode_probes_bit_exact(self):
        g = load_golden("codec")
        assert np.array_equal(oc.e4m3_encode(g["probes"]), g["encoded"])

    def test_known_answers(self):
        # test_numerics.py:46-60 spot values
        assert oc.e4m3_decode(0x7E) == 448.0 and oc.e4m3_decode(0x38) == 1.0
        assert oc.e4m3_decode(0x01) == 2.0 ** -9
        assert math.isnan(oc.e4m3_decode(0x7F)) and math.isnan(oc.e4m3_decode(0xFF))
        assert int(oc.e4m3_encode(np.array([1e9]))[0]) == 0x7E       # saturates, never NaN
        assert int(oc.e4m3_encode(np.array([-0.0]))[0]) == 0x80

    def test_matches_ml_dtypes_on_f32(self):
        ml = pytest.importorskip("ml_dtypes")
        x = np.random.default_rng(3).normal(0, 30, 20000).astype(np.float32)
        x = np.clip(x, -448, 448)
        ref = x.astype(ml.float8_e4m3fn).view(np.uint8)
        assert np.array_equal(oc.e4m3_encode(x.astype(np.float64)), ref)

    @pytest.mark.parametrize("depth,key", [(1, "gemm_d1"), (2, "gemm_d2")])
    def test_fp16_accumulator_gemm_bit_exact(self, depth, key):
        g = load_golden("codec")
        got, ovf, conv = oc.fp8_gemm_fp16acc(g["gemm_a"], g["gemm_b"], depth)
        assert np.array_equal(got, g[key])
        assert ovf == int(g[key + "_ovf"]) and conv == int(g[key + "_conv"])

    def test_fp32_accumulator_gemm_bit_exact(self):
        g = load_golden("codec")
        assert np.array_equal(oc.fp8_gemm_fp32acc(g["gemm_a"], g["gemm_b"]), g["gemm_f32"])

    def test_overflow_witness(self):
        # 64 x (448*448) at depth 2 overflows and saturates (test_mma.py:66-69)
        g = load_golden("codec")
        big = np.full((4, 64), 0x7E, dtype=np.uint8)
        got, ovf, _ = oc.fp8_gemm_fp16acc(big, big.T.copy(), 2)
        assert ovf == int(g["big_ovf"]) > 0
        assert np.array_equal(got, g["big_out"])

    def test_range_rule(self):
        # quantization.py:56-68 / test_quantization.py:29-50
        for p_r, v_r in [(448.0, 2.25), (224.0, 4.5), (112.0, 9.0)]:
            oc.RangeConfig(p_r, v_r, 2)
        with pytest.raises(oc.RangeConfigError):
            oc.RangeConfig(448.0, 448.0, 1)
        with pytest.raises(oc.RangeConfigError):
            oc.RangeConfig(448.0, 4.5, 2)
        oc.RangeConfig(448.0, 4.5, 1)


class TestQuantizerKAT:
    """Known-answer tests copied in spirit from test_quantization.py:56-171."""

    def test_int8_formula(self):
        codes, scale = oc.int_quantize(np.array([[63.5, -63.5]]), 8)
        assert scale == 0.5 and codes.tolist() == [[127, -127]]

    def test_int4_formula(self):
        codes, scale = oc.int_quantize(np.array([[7.0, -7.0]]), 4)
        assert scale == 1.0 and codes.tolist() == [[7, -7]]

    def test_zero_tile_sentinel(self):
        codes, scale = oc.int_quantize(np.zeros((3, 4)), 8)
        assert scale == 1.0 and not codes.any()

    def test_p_tile_max_one(self):
        codes, scale = oc.p_quantize(np.array([[1.0, 0.5]]), 224.0)
        assert scale == 1.0 / 224.0 and oc.e4m3_decode(codes[0, 0]) == 224.0

    def test_v_channel(self):
        codes, scales = oc.v_quantize(np.array([[9.0], [-9.0]]), 4.5)
        assert scales.tolist() == [2.0]
        assert oc.e4m3_decode(codes).ravel().tolist() == [4.5, -4.5]


# ------------------------------------------------------------------ whole path vs fixtures
@pytest.mark.parametrize("name", golden_cases())
def test_prepass_bit_exact_vs_reference(name):
    g = load_golden(name)
    cfg = cfg_from(g)
    for h in range(cfg.num_heads):
        qt = oc.prepass(g["q"][h], g["k"][h], g["v"][h], cfg)
        assert np.array_equal(qt.q_codes, g["q_codes"][h])
        assert np.array_equal(qt.q_scale, g["q_scale"][h])
        assert np.array_equal(qt.k_codes, g["k_codes"][h])
        assert np.array_equal(qt.k_scale, g["k_scale"][h])
        assert np.array_equal(qt.v_codes, g["v_codes"][h])
        assert np.array_equal(qt.v_scale, g["v_scale"][h])
        assert np.array_equal(qt.bias, g["bias"][h])
        assert np.array_equal(qt.q_mean, g["q_mean"][h])


@pytest.mark.parametrize("name", [n for n in golden_cases() if n != "attn_oracle"])
def test_attention_matches_reference_output(name):
    g = load_golden(name)
    cfg = cfg_from(g)
    rep = oc.attention_quantized(g["q"], g["k"], g["v"], cfg)
    np.testing.assert_allclose(rep.output, g["out"], rtol=0, atol=1e-12)
    assert rep.overflow_events == int(g["overflow"])
    assert rep.fp16_to_fp32_conversions == int(g["conversions"])
    assert rep.mma_invocations == int(g["mma"])
    assert rep.p_scale_min == float(g["p_scale_min"]) and rep.p_scale_max == float(g["p_scale_max"])
    exact = oc.attention_reference(g["q"], g["k"], g["v"], cfg)
    np.testing.assert_allclose(exact, g["out_exact"], rtol=0, atol=1e-12)


@pytest.mark.slow
def test_oracle_config_matches_reference_output():
    g = load_golden("attn_oracle")
    rep = oc.attention_quantized(g["q"], g["k"], g["v"], cfg_from(g))
    np.testing.assert_allclose(rep.output, g["out"], rtol=0, atol=1e-12)


def test_live_reference_on_fresh_seed(lpattn):
    """Where the reference exists, compare on inputs the fixtures never saw."""
    from lpattn.attention import AttentionConfig, attention_quantized
    rng = np.random.Generator(np.random.Philox(777))
    q, k, v = (rng.normal(size=(1, 160, 64)) for _ in range(3))
    ref = attention_quantized(q, k, v, AttentionConfig(seq_len=160, head_dim=64, causal=True))
    ours = oc.attention_quantized(q, k, v, oc.AttentionConfig(seq_len=160, head_dim=64, causal=True))
    np.testing.assert_allclose(ours.output, ref.output, rtol=0, atol=1e-12)
    assert ours.mma_invocations == ref.mma_invocations


@pytest.mark.parametrize("case", ["exact_ties", "huge_offsets", "zeros_subnormals", "tiny_blocks"])
def test_oracle_prepass_edges_vs_live_reference(lpattn, case):
    """The oracle's quantizers equal the reference's on the adversarial inputs the GPU prepass is
    tested with (tests/test_gpu_prepass_edges.py): ties, huge offsets, zeros, subnormals."""
    from lpattn import quantization as rq
    from edge_inputs import CASES
    q, k, v, smoothing = CASES[case]()
    h, n, d = q.shape
    cfg = oc.AttentionConfig(seq_len=n, head_dim=d, num_heads=h, smoothing=smoothing)
    for hh in range(h):
        ours = oc.prepass(q[hh], k[hh], v[hh], cfg)
        qs, ks = (rq.smooth_q(q[hh])[0], rq.smooth_k(k[hh])[0]) if smoothing else (
            q[hh].astype(np.float64), k[hh].astype(np.float64))
        npad = -(-n // 64) * 64
        ksp = np.zeros((npad, d))
        ksp[:n] = ks
        vp = np.zeros((npad, d))
        vp[:n] = v[hh]
        for j in range(npad // 64):
            kb = rq.quantize_int_block(ksp[j * 64:(j + 1) * 64])
            assert np.array_equal(ours.k_codes[j * 64:(j + 1) * 64], kb.codes) and ours.k_scale[j] == kb.scale
            vb = rq.quantize_v_per_channel(vp[j * 64:(j + 1) * 64], 4.5)
            assert np.array_equal(ours.v_codes[j * 64:(j + 1) * 64], vb.codes)
            assert np.array_equal(ours.v_scale[j], vb.scales)
        for i in range(-(-n // 128)):
            qb = rq.quantize_int_block(qs[i * 128:min((i + 1) * 128, n)])
            assert np.array_equal(ours.q_codes[i * 128:min((i + 1) * 128, n)], qb.codes)
            assert ours.q_scale[i] == qb.scale
