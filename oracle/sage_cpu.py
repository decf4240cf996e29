"""CPU restatement of the reference's quantized-attention path -- TEST INFRASTRUCTURE ONLY.

This module is the parity *checker* for the B200 kernels.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import it.
The product path (``paper_2505_21136_b200``) never imports it and has no CPU
fallback.

It restates, in numpy, the arithmetic of the reference simulator ``lpattn``
(``/root/reference/pkg/src/lpattn``).  Each function cites the reference
file:line it follows.  Parity of this restatement is PINNED two ways:

* ``tests/golden/*.npz`` -- fixtures produced by importing the unmodified
  reference (``tests/golden/make_golden.py``), checked bit-for-bit by
  ``tests/test_oracle_golden.py`` (runs on the GPU box, no reference needed);
* when ``/root/reference`` is importable (the build container), the same test
  module also runs the reference live on fresh seeded inputs.

Numerics mirrored exactly:
  * FP64 per-head channel means for Q and K smoothing (quantization.py:124-148)
  * symmetric INT8/INT4 quantization, RNE of x/scale in FP64 (quantization.py:151-160)
  * E4M3 "fn" saturating RNE encode (numerics.py:152-182)
  * per-(64-key block, channel) V scales with range v_r (quantization.py:178-188)
  * per-(128x64 tile) P scales with range p_r (quantization.py:163-175)
  * FP8 x FP8 -> FP16 sequential RNE accumulation in k-groups of 32, with
    depth-2 buffering and saturate-and-count overflow (mma.py:102-166)
  * FP32 sequential RNE accumulation baseline (mma.py:169-181)
  * the tiled online-softmax recurrence with causal and pad masking
    (attention.py:128-154, 232-316)
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

__all__ = [
    "FP16_MAX", "E4M3_MAX", "NEG_INF", "K_GROUP", "RANGE_PRODUCT_LIMIT",
    "RangeConfig", "RangeConfigError", "AttentionConfig", "RunReport",
    "e4m3_decode", "e4m3_encode", "fp16_round_sat",
    "int_quantize", "p_quantize", "v_quantize", "smooth",
    "fp8_gemm_fp16acc", "fp8_gemm_fp32acc",
    "QuantizedTensors", "prepass", "attention_quantized", "attention_reference",
    "compare", "MetricsReport",
]

FP16_MAX = 65504.0          # numerics.py:35
E4M3_MAX = 448.0            # numerics.py:37
NEG_INF = -1.0e30           # attention.py:55
K_GROUP = 32                # mma.py:49 (instruction k extent)
RANGE_PRODUCT_LIMIT = FP16_MAX / K_GROUP   # quantization.py:26 -> 2047.0


# --------------------------------------------------------------------------- E4M3
def _e4m3_value_of_code(code: int) -> float:
    """Field math for one E4M3 'fn' code (numerics.py:49-64)."""
    e = (code >> 3) & 0xF
    m = code & 0x7
    if e == 0xF and m == 0x7:
        return math.nan
    mag = m * 2.0 ** -9 if e == 0 else (8 + m) * 2.0 ** (e - 10)
    return -mag if code & 0x80 else mag


_E4M3_TABLE = np.array([_e4m3_value_of_code(c) for c in range(256)], dtype=np.float64)
# 0x00..0x7E are the non-negative finite codes, increasing in value.
_E4M3_POS = _E4M3_TABLE[:0x7F].copy()


def e4m3_decode(codes) -> np.ndarray:
    """Exact value of E4M3 codes (numerics.py:185-190)."""
    return _E4M3_TABLE[np.asarray(codes, dtype=np.uint8)]


def e4m3_encode(x) -> np.ndarray:
    """Round finite float64 values to E4M3 codes, RNE, saturating at +-448.

    Restates numerics.py:152-182 as a nearest-neighbour search on the sorted
    positive grid; ties go to the even code (= even mantissa LSB, since the
    positive codes are monotone in value).  -0 and negative values carry 0x80.
    """
    x = np.asarray(x, dtype=np.float64)
    if not np.all(np.isfinite(x)):
        raise ValueError("e4m3_encode requires finite input")
    mag = np.abs(x)
    hi = np.searchsorted(_E4M3_POS, mag, side="left")      # POS[hi-1] < mag <= POS[hi]
    hi = np.minimum(hi, 0x7E)
    lo = np.maximum(hi - 1, 0)
    d_lo = mag - _E4M3_POS[lo]
    d_hi = _E4M3_POS[hi] - mag
    pick_hi = (d_hi < d_lo) | ((d_hi == d_lo) & (hi % 2 == 0))
    code = np.where(pick_hi, hi, lo)
    code = np.where(mag >= E4M3_MAX, 0x7E, code)            # saturate
    code = np.where(mag == 0.0, 0, code)
    code = code.astype(np.uint8) | np.where(np.signbit(x), np.uint8(0x80), np.uint8(0))
    return code.astype(np.uint8)


# --------------------------------------------------------------------------- FP16
def fp16_round_sat(values: np.ndarray) -> tuple[np.ndarray, int]:
    """RNE to binary16, clamp overflow to +-65504 and count it (mma.py:102-113)."""
    with np.errstate(over="ignore"):
        h = np.asarray(values, dtype=np.float64).astype(np.float16)
    bad = np.isinf(h)
    n_bad = int(bad.sum())
    if n_bad:
        h = np.where(bad, np.copysign(np.float16(FP16_MAX), h), h).astype(np.float16)
    return h, n_bad


# --------------------------------------------------------------------------- ranges
class RangeConfigError(ValueError):
    """p_r * v_r exceeds the FP16 accumulator bound (quantization.py:29-30)."""


@dataclass(frozen=True)
class RangeConfig:
    """(p_r, v_r, depth) with the 2047/depth rule (quantization.py:33-68)."""

    p_r: float
    v_r: float
    buffering_depth: int = 2
    expect_overflow: bool = False

    def __post_init__(self):
        if not (self.p_r > 0 and self.v_r > 0):
            raise RangeConfigError("p_r and v_r must be positive")
        if self.buffering_depth not in (1, 2):
            raise RangeConfigError("buffering_depth must be 1 or 2")
        if not self.expect_overflow and self.p_r * self.v_r > RANGE_PRODUCT_LIMIT / self.buffering_depth:
            raise RangeConfigError(
                f"p_r*v_r = {self.p_r * self.v_r:g} > {RANGE_PRODUCT_LIMIT / self.buffering_depth:g}")


@dataclass(frozen=True)
class AttentionConfig:
    """Problem + pipeline knobs, defaults of attention.py:58-95."""

    seq_len: int
    head_dim: int
    num_heads: int = 1
    block_q: int = 128
    block_k: int = 64
    qk_bits: int = 8
    range: RangeConfig = field(default_factory=lambda: RangeConfig(224.0, 4.5, 2))
    causal: bool = False
    smoothing: bool = True
    softmax_scale: Optional[float] = None
    pv_accumulator: str = "fp16"

    @property
    def scale(self) -> float:
        return self.softmax_scale if self.softmax_scale is not None else 1.0 / math.sqrt(self.head_dim)


# --------------------------------------------------------------------------- quantizers
def smooth(x: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Subtract the FP64 per-channel token mean (quantization.py:124-148)."""
    x = np.asarray(x, dtype=np.float64)
    mu = x.mean(axis=0)
    return x - mu, mu


def int_quantize(x: np.ndarray, bits: int = 8) -> tuple[np.ndarray, float]:
    """Symmetric per-tile integer quantization (quantization.py:151-160).

    scale = max|x| / qmax (1.0 for an all-zero tile); codes = clip(rne(x/scale)).
    """
    qmax = (1 << (bits - 1)) - 1
    x = np.asarray(x, dtype=np.float64)
    peak = float(np.abs(x).max()) if x.size else 0.0
    scale = peak / qmax if peak > 0.0 else 1.0
    codes = np.clip(np.rint(x / scale), -qmax, qmax).astype(np.int32)
    return codes, scale


def p_quantize(p: np.ndarray, p_r: float) -> tuple[np.ndarray, float]:
    """One E4M3 scale for the whole score tile (quantization.py:163-175)."""
    peak = float(np.abs(p).max()) if p.size else 0.0
    scale = peak / p_r if peak > 0.0 else 1.0
    return e4m3_encode(p / scale), scale


def v_quantize(v: np.ndarray, v_r: float) -> tuple[np.ndarray, np.ndarray]:
    """One E4M3 scale per channel of a key block (quantization.py:178-188)."""
    v = np.asarray(v, dtype=np.float64)
    peaks = np.abs(v).max(axis=0) if v.shape[0] else np.zeros(v.shape[1])
    scales = np.where(peaks > 0.0, peaks / v_r, 1.0)
    return e4m3_encode(v / scales), scales


# --------------------------------------------------------------------------- emulated MMA
def fp8_gemm_fp16acc(a_codes: np.ndarray, b_codes: np.ndarray, depth: int = 2) -> tuple[np.ndarray, int, int]:
    """(M,K) x (K,N) E4M3 product through the FP16 accumulator (mma.py:116-166).

    Within each 32-wide k-group the exact products are folded into an FP16
    register one at a time in index order (one RNE per add).  With depth 2,
    consecutive group sums are combined in FP16 before the single FP32
    conversion.  Returns (fp32 result, overflow events, conversions).
    """
    a = e4m3_decode(a_codes)
    b = e4m3_decode(b_codes)
    m, kdim = a.shape
    n = b.shape[1]
    if kdim % K_GROUP:
        raise ValueError("k extent must be a multiple of 32")
    acc32 = np.zeros((m, n), dtype=np.float32)
    overflow = 0
    conversions = 0
    held = None
    for g0 in range(0, kdim, K_GROUP):
        reg = np.zeros((m, n), dtype=np.float16)
        for t in range(g0, g0 + K_GROUP):
            reg, bad = fp16_round_sat(reg.astype(np.float64) + np.outer(a[:, t], b[t]))
            overflow += bad
        if depth == 1:
            acc32 = acc32 + reg.astype(np.float32)
            conversions += m * n
        elif held is None:
            held = reg
        else:
            held, bad = fp16_round_sat(held.astype(np.float64) + reg.astype(np.float64))
            overflow += bad
            acc32 = acc32 + held.astype(np.float32)
            conversions += m * n
            held = None
    if held is not None:
        acc32 = acc32 + held.astype(np.float32)
        conversions += m * n
    return acc32, overflow, conversions


def fp8_gemm_fp32acc(a_codes: np.ndarray, b_codes: np.ndarray) -> np.ndarray:
    """Sequential FP32 RNE accumulation of exact products (mma.py:169-181)."""
    a = e4m3_decode(a_codes)
    b = e4m3_decode(b_codes)
    acc = np.zeros((a.shape[0], b.shape[1]), dtype=np.float32)
    for t in range(a.shape[1]):
        acc = (acc.astype(np.float64) + np.outer(a[:, t], b[t])).astype(np.float32)
    return acc


# --------------------------------------------------------------------------- prepass
@dataclass
class QuantizedTensors:
    """Everything the reference derives from Q/K/V before the tile loop, one head.

    Shapes follow the reference tiling (attention.py:259-281):
      q_codes (N, D) int8; q_scale (ceil(N/128),) f64
      k_codes (Np, D) int8 with Np = ceil(N/64)*64; k_scale (Np/64,) f64
      v_codes (Np, D) uint8 E4M3; v_scale (Np/64, D) f64
      bias (Np,) f64 = q_mean . Ks_j (zero when smoothing is off)
    """

    q_codes: np.ndarray
    q_scale: np.ndarray
    k_codes: np.ndarray
    k_scale: np.ndarray
    v_codes: np.ndarray
    v_scale: np.ndarray
    bias: np.ndarray
    k_smoothed: np.ndarray
    q_mean: np.ndarray
    k_mean: np.ndarray


def prepass(q: np.ndarray, k: np.ndarray, v: np.ndarray, cfg: AttentionConfig) -> QuantizedTensors:
    """Smooth, pad and quantize one head (attention.py:259-281, 288-289)."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    n, d = q.shape
    bq, bk = cfg.block_q, cfg.block_k
    if cfg.smoothing:
        qs, q_mean = smooth(q)
        ks, k_mean = smooth(k)
    else:
        qs, ks = q, k
        q_mean = np.zeros(d)
        k_mean = np.zeros(d)
    n_pad = -(-n // bk) * bk
    ks_p = np.zeros((n_pad, d))
    ks_p[:n] = ks
    v_p = np.zeros((n_pad, d))
    v_p[:n] = v
    nkb = n_pad // bk
    k_codes = np.zeros((n_pad, d), dtype=np.int8)
    v_codes = np.zeros((n_pad, d), dtype=np.uint8)
    k_scale = np.zeros(nkb)
    v_scale = np.zeros((nkb, d))
    for j in range(nkb):
        rows = slice(j * bk, (j + 1) * bk)
        c, s = int_quantize(ks_p[rows], cfg.qk_bits)
        k_codes[rows], k_scale[j] = c, s
        vc, vs = v_quantize(v_p[rows], cfg.range.v_r)
        v_codes[rows], v_scale[j] = vc, vs
    nqt = -(-n // bq)
    q_codes = np.zeros((n, d), dtype=np.int8)
    q_scale = np.zeros(nqt)
    for i in range(nqt):
        rows = slice(i * bq, min((i + 1) * bq, n))
        c, s = int_quantize(qs[rows], cfg.qk_bits)
        q_codes[rows], q_scale[i] = c, s
    bias = np.zeros(n_pad)
    if cfg.smoothing:
        for j in range(nkb):
            rows = slice(j * bk, (j + 1) * bk)
            bias[rows] = q_mean @ ks_p[rows].T     # same GEMV as attention.py:289
    return QuantizedTensors(q_codes, q_scale, k_codes, k_scale, v_codes, v_scale, bias,
                            ks_p, q_mean, k_mean)


# --------------------------------------------------------------------------- attention
@dataclass
class RunReport:
    """Mirror of attention.py:114-125."""

    output: np.ndarray
    overflow_events: int
    fp16_to_fp32_conversions: int
    mma_invocations: int
    p_scale_min: float
    p_scale_max: float
    v_scale_min: float
    v_scale_max: float


def _as_heads(x, cfg: AttentionConfig) -> np.ndarray:
    a = np.asarray(x, dtype=np.float64)
    if a.ndim == 2:
        a = a[None]
    if a.shape != (cfg.num_heads, cfg.seq_len, cfg.head_dim):
        raise ValueError(f"shape {a.shape} does not match config")
    if not np.isfinite(a).all():
        raise ValueError("Q/K/V must be finite")
    return a


def _n_visible(cfg: AttentionConfig, q_stop: int, nkb: int) -> int:
    """Causal visibility of key tiles (attention.py:180-183)."""
    return min(nkb, -(-q_stop // cfg.block_k)) if cfg.causal else nkb


@dataclass
class TileStats:
    overflow: int = 0
    conversions: int = 0
    mma: int = 0
    p_scales: list = field(default_factory=list)


def attention_tile(qt: QuantizedTensors, cfg: AttentionConfig, i: int, stats: TileStats | None = None) -> np.ndarray:
    """Output rows of query tile i of one head from its prepass tensors: the body of the reference's
    tile loop (attention.py:282-305).  Used by attention_quantized and, on sampled tiles of full-size
    heads, by the GPU parity tests."""
    n, d, bq, bk = cfg.seq_len, cfg.head_dim, cfg.block_q, cfg.block_k
    sm = cfg.scale
    depth = cfg.range.buffering_depth
    st = stats if stats is not None else TileStats()
    nkb = qt.k_codes.shape[0] // bk
    i0 = i * bq
    i1 = min(i0 + bq, n)
    rows = i1 - i0
    qc = qt.q_codes[i0:i1].astype(np.int64)
    m_run = np.full(rows, -np.inf)
    l_run = np.zeros(rows)
    o_run = np.zeros((rows, d))
    for j in range(_n_visible(cfg, i1, nkb)):
        j0, j1 = j * bk, (j + 1) * bk
        s_int = qc @ qt.k_codes[j0:j1].astype(np.int64).T
        st.mma += rows * bk * (-(-d // K_GROUP))
        s = s_int * (qt.q_scale[i] * qt.k_scale[j])
        if cfg.smoothing:
            s = s + qt.q_mean @ qt.k_smoothed[j0:j1].T
        s = s * sm
        if cfg.causal:
            qi = np.arange(i0, i1)[:, None]
            kj = np.arange(j0, j1)[None, :]
            s = np.where(kj > qi, NEG_INF, s)
        if j1 > n:
            s[:, n - j0:] = NEG_INF
        # online softmax (attention.py:136-154)
        m_new = np.maximum(m_run, s.max(axis=1))
        p = np.exp(s - m_new[:, None])
        alpha = np.exp(m_run - m_new)
        l_run = l_run * alpha + p.sum(axis=1)
        o_run = o_run * alpha[:, None]
        m_run = m_new
        p_codes, p_scale = p_quantize(p, cfg.range.p_r)
        st.p_scales.append(p_scale)
        if cfg.pv_accumulator == "fp16":
            pv, ov, cv = fp8_gemm_fp16acc(p_codes, qt.v_codes[j0:j1], depth)
            st.overflow += ov
            st.conversions += cv
        else:
            pv = fp8_gemm_fp32acc(p_codes, qt.v_codes[j0:j1])
        st.mma += rows * d * (bk // K_GROUP)
        o_run = o_run + pv.astype(np.float64) * (p_scale * qt.v_scale[j])
    l_safe = np.where(l_run == 0.0, 1.0, l_run)
    return o_run / l_safe[:, None]


def attention_quantized(q, k, v, cfg: AttentionConfig) -> RunReport:
    """The reference operator (attention.py:232-316), head by head."""
    if cfg.head_dim % K_GROUP or cfg.block_k % K_GROUP:
        raise ValueError("head_dim and block_k must be multiples of 32")
    squeeze = np.ndim(q) == 2
    q3, k3, v3 = (_as_heads(t, cfg) for t in (q, k, v))
    out = np.empty_like(q3)
    n, bq = cfg.seq_len, cfg.block_q
    st = TileStats()
    v_lo, v_hi = math.inf, -math.inf
    for h in range(cfg.num_heads):
        qt = prepass(q3[h], k3[h], v3[h], cfg)
        v_lo = min(v_lo, float(qt.v_scale.min()))
        v_hi = max(v_hi, float(qt.v_scale.max()))
        for i, i0 in enumerate(range(0, n, bq)):
            out[h, i0:min(i0 + bq, n)] = attention_tile(qt, cfg, i, st)
    return RunReport(out[0] if squeeze else out, st.overflow, st.conversions, st.mma,
                     min(st.p_scales), max(st.p_scales), v_lo, v_hi)


def attention_reference(q, k, v, cfg: AttentionConfig) -> np.ndarray:
    """FP64 tiled attention, the accuracy baseline (attention.py:186-220)."""
    squeeze = np.ndim(q) == 2
    q3, k3, v3 = (_as_heads(t, cfg) for t in (q, k, v))
    out = np.empty_like(q3)
    n, bq, bk = cfg.seq_len, cfg.block_q, cfg.block_k
    nkb = -(-n // bk)
    for h in range(cfg.num_heads):
        qh, kh = q3[h], k3[h]
        q_mean = None
        if cfg.smoothing:
            qh, q_mean = smooth(qh)
            kh, _ = smooth(kh)
        for i0 in range(0, n, bq):
            i1 = min(i0 + bq, n)
            m_run = np.full(i1 - i0, -np.inf)
            l_run = np.zeros(i1 - i0)
            o_run = np.zeros((i1 - i0, cfg.head_dim))
            for j in range(_n_visible(cfg, i1, nkb)):
                j0, j1 = j * bk, min((j + 1) * bk, n)
                s = qh[i0:i1] @ kh[j0:j1].T
                if q_mean is not None:
                    s = s + q_mean @ kh[j0:j1].T
                s = s * cfg.scale
                if cfg.causal:
                    s = np.where(np.arange(j0, j1)[None, :] > np.arange(i0, i1)[:, None], NEG_INF, s)
                m_new = np.maximum(m_run, s.max(axis=1))
                p = np.exp(s - m_new[:, None])
                alpha = np.exp(m_run - m_new)
                l_run = l_run * alpha + p.sum(axis=1)
                o_run = o_run * alpha[:, None] + p @ v3[h][j0:j1]
                m_run = m_new
            out[h, i0:i1] = o_run / np.where(l_run == 0.0, 1.0, l_run)[:, None]
    return out[0] if squeeze else out


# --------------------------------------------------------------------------- metrics
@dataclass(frozen=True)
class MetricsReport:
    cossim: float
    l1: float
    rmse: float


def compare(o_ref, o_test) -> MetricsReport:
    """Flattened cossim / relative L1 / RMSE in float64 (metrics.py:33-57)."""
    a = np.asarray(o_ref, dtype=np.float64).ravel()
    b = np.asarray(o_test, dtype=np.float64).ravel()
    if a.shape != b.shape or a.size == 0:
        raise ValueError("shape mismatch or empty")
    na, nb, l1d = np.sqrt(np.sum(a * a)), np.sqrt(np.sum(b * b)), np.sum(np.abs(a))
    if na == 0 or l1d == 0 or nb == 0:
        raise ValueError("degenerate metric denominator")
    diff = a - b
    return MetricsReport(float(np.sum(a * b) / (na * nb)), float(np.sum(np.abs(diff)) / l1d),
                         float(np.sqrt(np.mean(diff * diff))))
