"""Generate the golden fixtures under tests/golden/ by running the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [/root/reference/pkg/src]

The reference package ``lpattn`` is imported read-only from its source tree;
nothing is copied.  Each fixture holds seeded inputs plus what the reference
computes from them, so the GPU box (which has no reference) can check both
our numpy restatement (``oracle/sage_cpu.py``) and the CUDA kernels against
the reference's own numbers.

Quantized tensors are extracted by re-driving the reference's quantizers in
the order of ``attention.py:259-281`` because ``attention_quantized`` does not
return them.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = Path(sys.argv[1] if len(sys.argv) > 1 else "/root/reference/pkg/src")
sys.path.insert(0, str(REF_SRC))

from lpattn import numerics, mma, quantization, tensorio  # noqa: E402
from lpattn.attention import (  # noqa: E402
    AttentionConfig, _pad_keys, attention_quantized, attention_reference,
)
from lpattn.quantization import RangeConfig  # noqa: E402


def extract_quant(q3, k3, v3, cfg):
    """Re-drive the reference quantizers for every head (attention.py:259-281)."""
    out = {k: [] for k in ("q_codes", "q_scale", "k_codes", "k_scale", "v_codes",
                           "v_scale", "bias", "q_mean", "k_mean")}
    for h in range(cfg.num_heads):
        qh, kh, vh = (np.asarray(t[h], dtype=np.float64) for t in (q3, k3, v3))
        if cfg.smoothing:
            qh, q_mean = quantization.smooth_q(qh)
            kh, k_mean = quantization.smooth_k(kh)
        else:
            q_mean = np.zeros(cfg.head_dim)
            k_mean = np.zeros(cfg.head_dim)
        kh_p, vh_p, _ = _pad_keys(kh, vh, cfg.block_k)
        nkb = kh_p.shape[0] // cfg.block_k
        kc, ks, vc, vs, bias = [], [], [], [], []
        for j in range(nkb):
            rows = slice(j * cfg.block_k, (j + 1) * cfg.block_k)
            kb = quantization.quantize_int_block(kh_p[rows], cfg.qk_bits)
            vb = quantization.quantize_v_per_channel(vh_p[rows], cfg.range.v_r)
            kc.append(kb.codes)
            ks.append(kb.scale)
            vc.append(vb.codes)
            vs.append(vb.scales)
            bias.append(q_mean @ kh_p[rows].T if cfg.smoothing else np.zeros(cfg.block_k))
        qc, qs = [], []
        for i0 in range(0, cfg.seq_len, cfg.block_q):
            qb = quantization.quantize_int_block(qh[i0:i0 + cfg.block_q], cfg.qk_bits)
            qc.append(qb.codes)
            qs.append(qb.scale)
        out["q_codes"].append(np.concatenate(qc).astype(np.int8))
        out["q_scale"].append(np.array(qs))
        out["k_codes"].append(np.concatenate(kc).astype(np.int8))
        out["k_scale"].append(np.array(ks))
        out["v_codes"].append(np.concatenate(vc).astype(np.uint8))
        out["v_scale"].append(np.stack(vs))
        out["bias"].append(np.concatenate(bias))
        out["q_mean"].append(q_mean)
        out["k_mean"].append(k_mean)
    return {k: np.stack(v) for k, v in out.items()}


def philox(shape, seed, dist="gaussian", **kw):
    arr, _ = tensorio.generate(shape, dist, seed, **kw)
    return arr


def case(name, heads, seq, dim, *, seed=0, causal=False, dist="gaussian", v_offset=False,
         bf16=False, smoothing=True, qk_bits=8, pv="fp16", rng_cfg=(224.0, 4.5, 2, False),
         softmax_scale=None):
    shape = (heads, seq, dim)
    q = philox(shape, seed, dist)
    k = philox(shape, seed + 1, dist)
    v = philox(shape, seed + 2, dist)
    if v_offset:
        off = np.random.Generator(np.random.Philox(seed + 3)).normal(0.0, 2.0, size=(heads, 1, dim))
        v = (v + off).astype(np.float32)
    if bf16:  # round to bf16-representable float32 values (RNE on the top 16 bits)
        def to_bf16(a):
            u = a.view(np.uint32).astype(np.uint64)
            u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
            return u.astype(np.uint32).view(np.float32)
        q, k, v = to_bf16(q), to_bf16(k), to_bf16(v)
    p_r, v_r, depth, waive = rng_cfg
    cfg = AttentionConfig(seq_len=seq, head_dim=dim, num_heads=heads, causal=causal,
                          smoothing=smoothing, qk_bits=qk_bits, pv_accumulator=pv,
                          range=RangeConfig(p_r, v_r, depth, waive), softmax_scale=softmax_scale)
    rep = attention_quantized(q, k, v, cfg)
    ref = attention_reference(q, k, v, cfg)
    quant = extract_quant(q, k, v, cfg)
    np.savez_compressed(
        HERE / f"attn_{name}.npz", q=q, k=k, v=v,
        out=rep.output, out_exact=ref,
        overflow=rep.overflow_events, conversions=rep.fp16_to_fp32_conversions,
        mma=rep.mma_invocations, p_scale_min=rep.p_scale_min, p_scale_max=rep.p_scale_max,
        v_scale_min=rep.v_scale_min, v_scale_max=rep.v_scale_max,
        cfg=np.array([seq, dim, heads, int(causal), int(smoothing), qk_bits,
                      int(pv == "fp16"), depth, int(waive)]),
        ranges=np.array([p_r, v_r, -1.0 if softmax_scale is None else softmax_scale]),
        **quant,
    )
    print(f"attn_{name}: overflow={rep.overflow_events} mma={rep.mma_invocations}")


def codec_fixture():
    codes = np.arange(256, dtype=np.uint8)
    decoded = numerics.e4m3_decode(codes)
    pos = decoded[:0x7F]
    mids = (pos[1:] + pos[:-1]) / 2
    probes = np.concatenate([
        pos, mids, np.nextafter(mids, np.inf), np.nextafter(mids, -np.inf),
        np.array([0.0, -0.0, 448.0, 449.0, 463.99, 464.0, 464.01, 480.0, 1e6, 2.0 ** -10,
                  2.0 ** -10 + 1e-12, 3 * 2.0 ** -11, 1e-30]),
        np.random.Generator(np.random.Philox(7)).normal(0, 50, 4000),
        np.random.Generator(np.random.Philox(8)).uniform(-1, 1, 2000) * 2.0 ** -6,
    ])
    probes = np.concatenate([probes, -probes])
    enc = numerics.e4m3_encode(probes)
    rng = np.random.Generator(np.random.Philox(9))
    # FP16-accumulator GEMMs on random finite codes (no NaN codes)
    a = rng.integers(0, 0x7E, size=(16, 128)).astype(np.uint8) | (rng.integers(0, 2, (16, 128)) << 7).astype(np.uint8)
    b = rng.integers(0, 0x70, size=(128, 24)).astype(np.uint8) | (rng.integers(0, 2, (128, 24)) << 7).astype(np.uint8)
    g1, r1 = mma.gemm_emulated(a, b, "fp8_fp16acc", buffering_depth=1)
    g2, r2 = mma.gemm_emulated(a, b, "fp8_fp16acc", buffering_depth=2)
    g32, _ = mma.gemm_emulated(a, b, "fp8_fp32acc")
    big = np.full((4, 64), 0x7E, dtype=np.uint8)  # 448 x 448 -> overflow witness
    gbig, rbig = mma.gemm_emulated(big, big.T.copy(), "fp8_fp16acc", buffering_depth=2)
    np.savez_compressed(
        HERE / "codec.npz", decoded=decoded, probes=probes, encoded=enc,
        gemm_a=a, gemm_b=b, gemm_d1=g1, gemm_d2=g2, gemm_f32=g32,
        gemm_d1_conv=r1.fp16_to_fp32_conversions, gemm_d2_conv=r2.fp16_to_fp32_conversions,
        gemm_d1_ovf=r1.overflow.count, gemm_d2_ovf=r2.overflow.count,
        big_out=gbig, big_ovf=rbig.overflow.count,
    )
    print("codec: ok")


if __name__ == "__main__":
    codec_fixture()
    # configs[0] of BASELINE.json: the CPU oracle config, fp32 N(0,1), Philox seeds 0,1,2 (cli.py:161-163)
    case("oracle", 2, 1024, 64, seed=0)
    case("ragged_causal_d128", 1, 200, 128, seed=11, causal=True)
    case("ragged_voffset_d64", 2, 100, 64, seed=12, v_offset=True)
    case("uniform_d128", 1, 384, 128, seed=13, dist="uniform")
    case("bf16_d128", 2, 512, 128, seed=14, bf16=True)
    case("bf16_causal_d64", 1, 333, 64, seed=15, bf16=True, causal=True)
    case("nosmooth_d64", 1, 130, 64, seed=16, smoothing=False)
    case("int4_d64", 1, 256, 64, seed=17, qk_bits=4)
    case("fp32acc_d64", 1, 256, 64, seed=18, pv="fp32", rng_cfg=(448.0, 448.0, 1, True))
    case("depth1_d128", 1, 192, 128, seed=19, rng_cfg=(448.0, 4.5, 1, False))
    case("seq1_d64", 1, 1, 64, seed=20)
    case("scale_d128", 1, 256, 128, seed=21, softmax_scale=0.05, rng_cfg=(112.0, 9.0, 2, False))
    # head dims 32 (the reference's own test dim) and 96: zero-padded channels on the 64/128 kernels
    case("d32", 2, 256, 32, seed=22)
    case("ragged_causal_d96", 1, 200, 96, seed=23, causal=True)
