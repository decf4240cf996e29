"""ctypes binding of the C ABI in include/sa2pp.h (the same stub INTEGRATION.md shows).

The library is loaded from this package directory (built in-tree by build.py).
There is no fallback: if the library or a GPU is missing, calls raise.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libsa2pp.so"
if os.environ.get("SA2PP_LIB"):  # development A/B of library builds (tools/build_variant.py)
    LIB_PATH = Path(os.environ["SA2PP_LIB"]).resolve()

SA2PP_OK, SA2PP_ERR_INVALID, SA2PP_ERR_UNSUPPORTED, SA2PP_ERR_RANGE, SA2PP_ERR_CUDA = range(5)
SA2PP_F32, SA2PP_F16, SA2PP_BF16 = range(3)
SA2PP_ACC_F16, SA2PP_ACC_F32 = range(2)

EXPORTED = (
    "sa2pp_version", "sa2pp_last_error", "sa2pp_check_problem", "sa2pp_quant_sizes",
    "sa2pp_prepass", "sa2pp_attn_fwd", "sa2pp_sageattn", "sa2pp_set_debug_buffer",
    "sa2pp_set_trace_buffer", "sa2pp_host_pipeline_create", "sa2pp_host_pipeline_run",
    "sa2pp_host_pipeline_sync", "sa2pp_host_pipeline_destroy", "sa2pp_host_pipeline_run_report",
    "sa2pp_analytic_counts", "sa2pp_report_init", "sa2pp_attn_fwd_units",
)


class Problem(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("heads_q", C.c_int32), ("heads_kv", C.c_int32),
        ("seq_len", C.c_int32), ("head_dim", C.c_int32), ("causal", C.c_int32),
        ("smoothing", C.c_int32), ("qk_bits", C.c_int32), ("pv_accum", C.c_int32),
        ("buffering_depth", C.c_int32), ("expect_overflow", C.c_int32),
        ("sm_scale", C.c_double), ("p_r", C.c_double), ("v_r", C.c_double),
    ]


class Inputs(C.Structure):
    _fields_ = [
        ("dtype", C.c_int), ("q", C.c_void_p), ("k", C.c_void_p), ("v", C.c_void_p),
        ("q_stride", C.c_int64 * 3), ("k_stride", C.c_int64 * 3), ("v_stride", C.c_int64 * 3),
    ]


class Quant(C.Structure):
    _fields_ = [(name, C.c_void_p) for name in (
        "q_codes", "q_scale", "q_scale64", "k_codes", "v_codes", "kv_meta", "kv_scale64",
        "bias", "bias_l2", "means")]


class QuantSizes(C.Structure):
    _fields_ = [(name, C.c_size_t) for name in (
        "q_codes", "q_scale", "q_scale64", "k_codes", "v_codes", "kv_meta", "kv_scale64",
        "bias", "bias_l2", "means", "workspace")]


class Output(C.Structure):
    _fields_ = [("dtype", C.c_int), ("o", C.c_void_p), ("o_stride", C.c_int64 * 3)]


class Report(C.Structure):
    _fields_ = [("overflow_events", C.c_uint32), ("p_scale_min_bits", C.c_uint32),
                ("p_scale_max_bits", C.c_uint32), ("reserved", C.c_uint32),
                ("v_scale_min_bits", C.c_uint64), ("v_scale_max_bits", C.c_uint64)]


class RunReport(C.Structure):  # sa2pp_run_report
    _fields_ = [("overflow_events", C.c_uint64), ("fp16_to_fp32_conversions", C.c_uint64),
                ("mma_invocations", C.c_uint64), ("p_scale_min", C.c_double), ("p_scale_max", C.c_double),
                ("v_scale_min", C.c_double), ("v_scale_max", C.c_double)]


_lib = None


def lib() -> C.CDLL:
    """Load libsa2pp.so once; raise loudly when it is absent (no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2505_21136_b200.build` "
                "(or __graft_entry__.build()); there is no CPU fallback")
        h = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_LOCAL)
        P = C.POINTER
        h.sa2pp_version.restype = C.c_int
        h.sa2pp_last_error.restype = C.c_char_p
        h.sa2pp_check_problem.argtypes = [P(Problem)]
        h.sa2pp_quant_sizes.argtypes = [P(Problem), P(QuantSizes)]
        h.sa2pp_prepass.argtypes = [P(Problem), P(Inputs), P(Quant), C.c_void_p, C.c_size_t, C.c_void_p]
        h.sa2pp_attn_fwd.argtypes = [P(Problem), P(Quant), P(Output), C.c_void_p, C.c_void_p]
        h.sa2pp_attn_fwd_units.argtypes = [P(Problem), P(Quant), P(Output), C.c_void_p, C.c_int64, C.c_int64,
                                           C.c_void_p]
        h.sa2pp_sageattn.argtypes = [P(Problem), P(Inputs), P(Quant), C.c_void_p, C.c_size_t,
                                     P(Output), C.c_void_p, C.c_void_p]
        h.sa2pp_set_debug_buffer.argtypes = [C.c_void_p]
        h.sa2pp_set_trace_buffer.argtypes = [C.c_void_p]
        h.sa2pp_host_pipeline_create.argtypes = [P(Problem), C.c_int, C.c_int, C.c_int, P(C.c_void_p)]
        h.sa2pp_host_pipeline_run.argtypes = [C.c_void_p] * 6
        h.sa2pp_host_pipeline_sync.argtypes = [C.c_void_p]
        h.sa2pp_host_pipeline_destroy.argtypes = [C.c_void_p]
        h.sa2pp_host_pipeline_run_report.argtypes = [C.c_void_p] * 5 + [P(RunReport)]
        h.sa2pp_analytic_counts.argtypes = [P(Problem), P(C.c_uint64), P(C.c_uint64)]
        h.sa2pp_report_init.argtypes = [C.c_void_p, C.c_void_p]
        for name in EXPORTED[2:]:
            getattr(h, name).restype = C.c_int
        _lib = h
    return _lib


class Sa2ppError(RuntimeError):
    pass


def check(rc: int) -> None:
    """Map a C status onto the reference's exception types (ValueError for bad input)."""
    if rc == SA2PP_OK:
        return
    msg = lib().sa2pp_last_error().decode()
    if rc in (SA2PP_ERR_INVALID, SA2PP_ERR_UNSUPPORTED):
        raise ValueError(msg)
    if rc == SA2PP_ERR_RANGE:
        from .config import RangeConfigError
        raise RangeConfigError(msg)
    raise Sa2ppError(msg)
