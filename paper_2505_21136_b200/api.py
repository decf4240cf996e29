"""Host API: `sageattn` (north-star drop-in) and `attention_quantized` (reference mirror).

Both run the sm_100a kernels through the C ABI (include/sa2pp.h).  PyTorch is
only the device-memory and stream plumbing; all arithmetic of the path runs in
the CUDA library.  There is no CPU fallback.
"""

from __future__ import annotations

import warnings

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _abi as A
from .config import AttentionConfig

_DT = {torch.float32: A.SA2PP_F32, torch.float16: A.SA2PP_F16, torch.bfloat16: A.SA2PP_BF16}


@dataclass
class QuantizedTensors:
    """Device tensors written by the prepass; layouts documented in include/sa2pp.h."""

    q_codes: torch.Tensor      # int8  [B, Hq, Nq_pad, D]
    q_scale: torch.Tensor      # f32   [B, Hq, nQT]
    q_scale64: torch.Tensor    # f64   [B, Hq, nQT]
    k_codes: torch.Tensor      # int8  [B, Hkv, Np, D]
    v_codes: torch.Tensor      # uint8 [B, Hkv, D, Np] (E4M3, channel-major)
    kv_meta: torch.Tensor      # f32   [B, Hkv, nKB, 4 + D]
    kv_scale64: torch.Tensor   # f64   [B, Hkv, nKB, 1 + D]
    bias: torch.Tensor         # f32   [B, Hq, Np]
    bias_l2: torch.Tensor      # f32   [B, Hq, Np]
    means: torch.Tensor        # f64   [B, Hq + Hkv, D]
    workspace: torch.Tensor    # u8 scratch

    @property
    def k_scale64(self) -> torch.Tensor:
        return self.kv_scale64[..., 0]

    @property
    def v_scale64(self) -> torch.Tensor:
        return self.kv_scale64[..., 1:]

    def struct(self) -> A.Quant:
        return A.Quant(*(t.data_ptr() for t in (
            self.q_codes, self.q_scale, self.q_scale64, self.k_codes, self.v_codes, self.kv_meta,
            self.kv_scale64, self.bias, self.bias_l2, self.means)))


def _problem(B, Hq, Hkv, N, D, *, causal, smoothing=True, qk_bits=8, pv_accum="fp16", depth=2,
             expect_overflow=False, sm_scale=None, p_r=224.0, v_r=4.5) -> A.Problem:
    return A.Problem(B, Hq, Hkv, N, D, int(bool(causal)), int(bool(smoothing)), qk_bits,
                     A.SA2PP_ACC_F16 if pv_accum == "fp16" else A.SA2PP_ACC_F32, depth,
                     int(bool(expect_overflow)), float("nan") if sm_scale is None else float(sm_scale),
                     float(p_r), float(v_r))


def padded_dim(d: int) -> int:
    """Kernel channel width for head_dim d (sa2pp_internal.h padded_dim): 32 -> 64, 96 -> 128."""
    return 64 if d <= 64 else 128


def alloc_quant(prob: A.Problem, device) -> QuantizedTensors:
    sz = A.QuantSizes()
    A.check(A.lib().sa2pp_quant_sizes(C_ref(prob), C_ref(sz)))
    B, Hq, Hkv, N = prob.batch, prob.heads_q, prob.heads_kv, prob.seq_len
    D = padded_dim(prob.head_dim)  # the kernels' channel width: head dims 32 / 96 run zero-padded
    n_qt, n_kb = -(-N // 128), -(-N // 64)
    nq_pad, np_ = n_qt * 128, n_kb * 64
    e = lambda *shape, dt: torch.empty(shape, dtype=dt, device=device)  # noqa: E731
    return QuantizedTensors(
        q_codes=e(B, Hq, nq_pad, D, dt=torch.int8),
        q_scale=e(B, Hq, n_qt, dt=torch.float32),
        q_scale64=e(B, Hq, n_qt, dt=torch.float64),
        k_codes=e(B, Hkv, np_, D, dt=torch.int8),
        v_codes=e(B, Hkv, D, np_, dt=torch.uint8),
        kv_meta=e(B, Hkv, n_kb, 4 + D, dt=torch.float32),
        kv_scale64=e(B, Hkv, n_kb, 1 + D, dt=torch.float64),
        bias=e(B, Hq, np_, dt=torch.float32),
        bias_l2=e(B, Hq, np_, dt=torch.float32),
        means=e(B, Hq + Hkv, D, dt=torch.float64),
        workspace=e(max(int(sz.workspace), 16), dt=torch.uint8),
    )


def C_ref(x):
    import ctypes
    return ctypes.byref(x)


def _bhnd_view(x: torch.Tensor, layout: str):
    """(B, H, N, D, strides(b, h, n)) for an HND [B,H,N,D] or NHD [B,N,H,D] tensor."""
    if x.dim() != 4:
        raise ValueError(f"expected a 4-D tensor, got shape {tuple(x.shape)}")
    if x.stride(-1) != 1:
        raise ValueError("the head_dim axis must be contiguous")
    if layout == "HND":
        B, H, N, D = x.shape
        return B, H, N, D, (x.stride(0), x.stride(1), x.stride(2))
    if layout == "NHD":
        B, N, H, D = x.shape
        return B, H, N, D, (x.stride(0), x.stride(2), x.stride(1))
    raise ValueError(f"tensor_layout must be 'HND' or 'NHD', got {layout!r}")


def _stream_ptr(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def sageattn(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, tensor_layout: str = "HND",
             is_causal: bool = False, sm_scale: Optional[float] = None, *, pv_accum: str = "fp16",
             smooth: bool = True, qk_bits: int = 8, p_r: float = 224.0, v_r: float = 4.5,
             buffering_depth: int = 2, expect_overflow: bool = False,
             out: Optional[torch.Tensor] = None, return_quant: bool = False,
             report: Optional[torch.Tensor] = None, quant: Optional[QuantizedTensors] = None,
             stream=None):
    """SageAttention2++ forward on B200.

    q: [B, Hq, N, D] (HND) or [B, N, Hq, D] (NHD); k, v: same with Hkv heads (Hq % Hkv == 0).
    dtype float16 / bfloat16 / float32, CUDA.  Returns o with q's shape, layout and dtype.
    Keyword-only extras: ``pv_accum="fp32"`` selects the SageAttention2 FP32-accumulator
    baseline, ``return_quant=True`` also returns the prepass tensors for bit-exact checks.
    """
    if not (q.is_cuda and k.is_cuda and v.is_cuda):
        raise ValueError("sageattn runs on CUDA tensors only (no CPU fallback)")
    if not (q.dtype == k.dtype == v.dtype) or q.dtype not in _DT:
        raise ValueError("q, k, v must share one dtype among float16, bfloat16, float32")
    B, Hq, N, D, qs = _bhnd_view(q, tensor_layout)
    Bk, Hkv, Nk, Dk, ks = _bhnd_view(k, tensor_layout)
    Bv, Hv, Nv, Dv, vs = _bhnd_view(v, tensor_layout)
    if (Bk, Nk, Dk) != (B, N, D) or (Bv, Hv, Nv, Dv) != (Bk, Hkv, Nk, Dk):
        raise ValueError(f"Q/K/V shapes disagree: {tuple(q.shape)}, {tuple(k.shape)}, {tuple(v.shape)}")
    prob = _problem(B, Hq, Hkv, N, D, causal=is_causal, smoothing=smooth, qk_bits=qk_bits,
                    pv_accum=pv_accum, depth=buffering_depth, expect_overflow=expect_overflow,
                    sm_scale=sm_scale, p_r=p_r, v_r=v_r)
    A.check(A.lib().sa2pp_check_problem(C_ref(prob)))
    qt = quant if quant is not None else alloc_quant(prob, q.device)
    if out is None:
        out = torch.empty_like(q)
    B_, Ho, No, Do, os_ = _bhnd_view(out, tensor_layout)
    if (B_, Ho, No, Do) != (B, Hq, N, D) or out.dtype not in _DT:
        raise ValueError("out must match q's shape")
    ins = A.Inputs(_DT[q.dtype], q.data_ptr(), k.data_ptr(), v.data_ptr(),
                   (A.C.c_int64 * 3)(*qs), (A.C.c_int64 * 3)(*ks), (A.C.c_int64 * 3)(*vs))
    o = A.Output(_DT[out.dtype], out.data_ptr(), (A.C.c_int64 * 3)(*os_))
    qs_struct = qt.struct()
    rep_ptr = report.data_ptr() if report is not None else None
    with torch.cuda.device(q.device):
        A.check(A.lib().sa2pp_sageattn(C_ref(prob), C_ref(ins), C_ref(qs_struct), qt.workspace.data_ptr(),
                                       qt.workspace.numel(), C_ref(o), rep_ptr, _stream_ptr(stream)))
    return (out, qt) if return_quant else out


class HostPipeline:
    """`sageattn` on pinned HOST tensors with the copies overlapped with the kernels.

    A thin owner of the native handle `sa2pp_host_pipeline_*` (csrc/host_pipeline.cu): the
    (batch, kv-head) units are cut into `chunks` (whole GQA groups, so every chunk is an
    independent attention problem: smoothing statistics are per head); chunk i's host->device
    copy, prepass + attention and device->host copy run on three native streams through a ring
    of `depth` device buffer sets that persists across calls, so PCIe traffic in both
    directions overlaps the tensor cores and consecutive calls overlap each other.
    Inputs [B, H, N, D] (HND, contiguous, pinned); the output is written into `out` (pinned) and
    is complete once the caller's current stream reaches the point after the call.  Inputs must
    be ready when called (the uploads do not wait for earlier work on the caller's stream).
    """

    def __init__(self, B, Hq, Hkv, N, D, dtype=torch.bfloat16, device="cuda", *, is_causal=False,
                 sm_scale=None, pv_accum="fp16", chunks=8, depth=3, **kw):
        if Hq % Hkv:
            raise ValueError("heads_q must be a multiple of heads_kv")
        if dtype not in _DT:
            raise ValueError("dtype must be float16, bfloat16 or float32")
        self.B, self.Hq, self.Hkv, self.N, self.D, self.dtype = B, Hq, Hkv, N, D, dtype
        self.device = torch.device(device)
        if self.device.index is None:
            self.device = torch.device("cuda", torch.cuda.current_device())
        prob = _problem(B, Hq, Hkv, N, D, causal=is_causal, pv_accum=pv_accum, sm_scale=sm_scale,
                        smoothing=kw.get("smooth", True), qk_bits=kw.get("qk_bits", 8),
                        p_r=kw.get("p_r", 224.0), v_r=kw.get("v_r", 4.5), depth=kw.get("buffering_depth", 2),
                        expect_overflow=kw.get("expect_overflow", False))
        self._h = A.C.c_void_p()
        with torch.cuda.device(self.device):
            A.check(A.lib().sa2pp_host_pipeline_create(C_ref(prob), _DT[dtype], chunks, depth, A.C.byref(self._h)))

    def __call__(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        B, Hq, Hkv, N, D = self.B, self.Hq, self.Hkv, self.N, self.D
        for t, h in ((q, Hq), (k, Hkv), (v, Hkv), (out, Hq)):
            if t.is_cuda or tuple(t.shape) != (B, h, N, D) or not t.is_contiguous() or t.dtype != self.dtype:
                raise ValueError("HostPipeline takes contiguous [B, H, N, D] host tensors of its dtype")
        caller = torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            A.check(A.lib().sa2pp_host_pipeline_run(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                                    out.data_ptr(), caller.cuda_stream))
        return out

    def run_report(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, out: torch.Tensor) -> A.RunReport:
        """Blocking call with the instrumented kernels; returns the reference's RunReport counters
        (sa2pp_host_pipeline_run_report) and leaves the output in `out`."""
        for t, h in ((q, self.Hq), (k, self.Hkv), (v, self.Hkv), (out, self.Hq)):
            if t.is_cuda or tuple(t.shape) != (self.B, h, self.N, self.D) or not t.is_contiguous() or t.dtype != self.dtype:
                raise ValueError("HostPipeline takes contiguous [B, H, N, D] host tensors of its dtype")
        rep = A.RunReport()
        with torch.cuda.device(self.device):
            A.check(A.lib().sa2pp_host_pipeline_run_report(self._h, q.data_ptr(), k.data_ptr(), v.data_ptr(),
                                                           out.data_ptr(), A.C.byref(rep)))
        return rep

    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            A.lib().sa2pp_host_pipeline_destroy(self._h)
            self._h = A.C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sageattn_host(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, is_causal: bool = False,
                  sm_scale: Optional[float] = None, *, out: Optional[torch.Tensor] = None, chunks: int = 8,
                  **kw) -> torch.Tensor:
    """One-shot `HostPipeline` call: pinned HND host tensors in, pinned host output out."""
    B, Hq, N, D = q.shape
    pipe = HostPipeline(B, Hq, k.shape[1], N, D, q.dtype, is_causal=is_causal, sm_scale=sm_scale, chunks=chunks,
                        **kw)
    if out is None:
        out = torch.empty(q.shape, dtype=q.dtype, pin_memory=True)
    return pipe(q, k, v, out)


def new_report(device) -> torch.Tensor:
    """Device RunReport buffer (sa2pp_report, 32 bytes): overflow count, min/max delta_P as float
    bits, min/max delta_V as double bits."""
    r = torch.zeros(8, dtype=torch.int32, device=device)
    r[1] = 0x7F800000  # +inf bits for the running minimum of delta_P
    r.view(torch.int64)[2] = 0x7FF0000000000000  # +inf bits (double) for the minimum of delta_V
    return r


def read_report(rep: torch.Tensor) -> dict:
    """Decode a device sa2pp_report (new_report) into the reference's field names."""
    raw = rep.cpu().numpy()
    u32, f32, f64 = raw.view(np.uint32), raw.view(np.float32), raw.view(np.float64)
    return {"overflow_events": int(u32[0]), "p_scale_min": float(f32[1]), "p_scale_max": float(f32[2]),
            "v_scale_min": float(f64[2]), "v_scale_max": float(f64[3])}


# ----------------------------------------------------------------------------- reference mirror
@dataclass
class RunReport:
    """Mirror of lpattn's RunReport (attention.py:114-125), produced on the GPU."""

    output: np.ndarray
    overflow_events: int
    fp16_to_fp32_conversions: int
    mma_invocations: int
    p_scale_min: float
    p_scale_max: float
    v_scale_min: float
    v_scale_max: float


def _visible(cfg: AttentionConfig, i_stop: int, n_kt: int) -> int:
    return min(n_kt, -(-i_stop // cfg.block_k)) if cfg.causal else n_kt


def _analytic_counts(cfg: AttentionConfig) -> tuple[int, int]:
    """(fp16->fp32 conversions, mma invocations) exactly as the reference counts them (mma.py:67-86)."""
    n, d, bq, bk = cfg.seq_len, cfg.head_dim, cfg.block_q, cfg.block_k
    n_kt = -(-n // bk)
    conv = mma = 0
    for i0 in range(0, n, bq):
        rows = min(bq, n - i0)
        vis = _visible(cfg, min(i0 + bq, n), n_kt)
        mma += vis * (rows * bk * (-(-d // MMA_K)) + rows * d * (bk // MMA_K))
        if cfg.pv_accumulator == "fp16":
            groups = bk // MMA_K
            per = -(-groups // cfg.range.buffering_depth)
            conv += vis * rows * d * per
    return conv * cfg.num_heads, mma * cfg.num_heads


MMA_K = 32


def attention_quantized(q, k, v, config: AttentionConfig, *, device: str = "cuda") -> RunReport:
    """Drop-in for lpattn.attention.attention_quantized (attention.py:232-316), on the B200.

    Accepts (seq, dim) or (heads, seq, dim) arrays like the reference; computes with the
    sm_100a kernels on float32 copies; returns the output as float64 with the same counters.
    """
    if config.head_dim % MMA_K != 0:
        raise ValueError(f"head_dim must be a multiple of {MMA_K} for the FP8 path")
    if config.block_k % MMA_K != 0:
        raise ValueError(f"block_k must be a multiple of {MMA_K} for the FP8 path")
    if (config.block_q, config.block_k) != (128, 64):
        raise ValueError("the B200 kernels are built for block_q=128, block_k=64 (reference defaults)")
    arrs = [np.asarray(t, dtype=np.float64) for t in (q, k, v)]
    if not (arrs[0].shape == arrs[1].shape == arrs[2].shape):
        raise ValueError(f"Q/K/V shapes disagree: {arrs[0].shape}, {arrs[1].shape}, {arrs[2].shape}")
    squeeze = arrs[0].ndim == 2
    if squeeze:
        arrs = [a[None] for a in arrs]
    if arrs[0].ndim != 3:
        raise ValueError("tensors must be (seq, dim) or (heads, seq, dim)")
    expected = (config.num_heads, config.seq_len, config.head_dim)
    if arrs[0].shape != expected:
        raise ValueError(f"tensor shape {arrs[0].shape} does not match config {expected}")
    if not all(np.isfinite(a).all() for a in arrs):
        raise ValueError("Q/K/V must be finite")
    a32 = [a.astype(np.float32) for a in arrs]
    if any(not np.array_equal(x.astype(np.float64), a) for x, a in zip(a32, arrs)):
        # the kernels read float32/16-bit inputs: quantized tensors are then bit-exact with the
        # reference run on the float32-rounded inputs, and the output within tolerance of this one
        warnings.warn("attention_quantized: float64 inputs are not float32-representable and are rounded to "
                      "float32 for the sm_100a path", RuntimeWarning, stacklevel=2)
    tq, tk, tv = (torch.from_numpy(a)[None].to(device) for a in a32)
    rep = new_report(tq.device)
    out, qt = sageattn(
        tq, tk, tv, "HND", config.causal, config.scale, pv_accum=config.pv_accumulator,
        smooth=config.smoothing, qk_bits=config.qk_bits, p_r=config.range.p_r, v_r=config.range.v_r,
        buffering_depth=config.range.buffering_depth, expect_overflow=config.range.expect_overflow,
        return_quant=True, report=rep)
    torch.cuda.synchronize(tq.device)
    r = read_report(rep)
    conv, mma = _analytic_counts(config)
    o = out[0].double().cpu().numpy()
    return RunReport(output=o[0] if squeeze else o, fp16_to_fp32_conversions=conv, mma_invocations=mma, **r)


def quantize(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, tensor_layout: str = "HND", *,
             smooth: bool = True, qk_bits: int = 8, v_r: float = 4.5, sm_scale: Optional[float] = None,
             stream=None) -> QuantizedTensors:
    """Run only the prepass (smoothing + INT8/E4M3 quantization) and return its tensors."""
    B, Hq, N, D, qs = _bhnd_view(q, tensor_layout)
    _, Hkv, _, _, ks = _bhnd_view(k, tensor_layout)
    _, _, _, _, vs = _bhnd_view(v, tensor_layout)
    prob = _problem(B, Hq, Hkv, N, D, causal=False, smoothing=smooth, qk_bits=qk_bits, v_r=v_r,
                    sm_scale=sm_scale)
    qt = alloc_quant(prob, q.device)
    ins = A.Inputs(_DT[q.dtype], q.data_ptr(), k.data_ptr(), v.data_ptr(),
                   (A.C.c_int64 * 3)(*qs), (A.C.c_int64 * 3)(*ks), (A.C.c_int64 * 3)(*vs))
    qs_struct = qt.struct()
    with torch.cuda.device(q.device):
        A.check(A.lib().sa2pp_prepass(C_ref(prob), C_ref(ins), C_ref(qs_struct), qt.workspace.data_ptr(),
                                      qt.workspace.numel(), _stream_ptr(stream)))
    return qt


def compare(o_ref, o_test):
    """cossim / relative L1 / RMSE in float64, as lpattn.metrics.compare (metrics.py:33-57)."""
    a = np.asarray(o_ref, dtype=np.float64).ravel()
    b = np.asarray(o_test, dtype=np.float64).ravel()
    if a.shape != b.shape or a.size == 0:
        raise ValueError("shape mismatch or empty tensors")
    na, nb, sa = math.sqrt(float(np.sum(a * a))), math.sqrt(float(np.sum(b * b))), float(np.sum(np.abs(a)))
    if na == 0.0 or sa == 0.0 or nb == 0.0:
        raise ValueError("degenerate metric denominator")
    d = a - b
    return float(np.sum(a * b)) / (na * nb), float(np.sum(np.abs(d))) / sa, math.sqrt(float(np.mean(d * d)))
