"""C-ABI and host-logic checks that need no GPU.

* libsa2pp.so loads and exports every function include/sa2pp.h declares;
* sa2pp_check_problem / sa2pp_quant_sizes apply the reference's validation rules
  (attention.py:74-85, 242-245; quantization.py:49-60) with the documented status codes;
* the Python mirror of AttentionConfig / RangeConfig behaves like the reference's;
* the product path refuses to run without CUDA (no silent CPU fallback).
"""

import ctypes
import re
from pathlib import Path

import pytest
import torch

import paper_2505_21136_b200 as sa
from paper_2505_21136_b200 import _abi as A
from paper_2505_21136_b200.api import _problem

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    text = (ROOT / "include" / "sa2pp.h").read_text()
    return sorted(set(re.findall(r"SA2PP_API\s+[\w\s\*]+?\b(sa2pp_\w+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(A.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = A.lib()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.sa2pp_version() == 100


def rc(**kw):
    base = dict(B=1, Hq=2, Hkv=2, N=1024, D=64)
    base.update({k: kw.pop(k) for k in list(kw) if k in base})
    prob = _problem(base["B"], base["Hq"], base["Hkv"], base["N"], base["D"], causal=False, **kw)
    return A.lib().sa2pp_check_problem(ctypes.byref(prob))


def test_valid_problem():
    assert rc() == A.SA2PP_OK
    assert rc(D=128, Hq=32, Hkv=8) == A.SA2PP_OK
    assert rc(N=1) == A.SA2PP_OK and rc(N=17776) == A.SA2PP_OK
    assert rc(D=32) == A.SA2PP_OK and rc(D=96, Hq=4, Hkv=2) == A.SA2PP_OK  # zero-padded to 64 / 128


def test_quant_sizes_of_padded_head_dims():
    """head_dim 32 / 96 quantize into the 64 / 128-channel layout the kernels read."""
    for d, dp in ((32, 64), (96, 128)):
        prob = _problem(1, 2, 2, 1000, d, causal=False)
        sz = A.QuantSizes()
        assert A.lib().sa2pp_quant_sizes(ctypes.byref(prob), ctypes.byref(sz)) == 0
        assert sz.k_codes == 2 * 16 * 64 * dp and sz.means == 2 * 2 * dp * 8
        assert sz.kv_scale64 == 2 * 16 * (1 + dp) * 8


@pytest.mark.parametrize("kw,code", [
    (dict(D=48), A.SA2PP_ERR_INVALID),            # not a multiple of 32 (attention.py:242-243)
    (dict(D=160), A.SA2PP_ERR_UNSUPPORTED),       # valid for the reference, not built here
    (dict(Hq=6, Hkv=4), A.SA2PP_ERR_INVALID),     # GQA group must divide
    (dict(N=0), A.SA2PP_ERR_INVALID),
    (dict(qk_bits=6), A.SA2PP_ERR_INVALID),       # attention.py:82-83
    (dict(p_r=448.0, v_r=448.0), A.SA2PP_ERR_RANGE),          # 2047/depth rule
    (dict(p_r=448.0, v_r=4.5, depth=2), A.SA2PP_ERR_RANGE),   # 2016 > 1023.5
    (dict(depth=3), A.SA2PP_ERR_RANGE),
])
def test_invalid_problems(kw, code):
    assert rc(**kw) == code
    assert A.lib().sa2pp_last_error()


def test_range_waiver_and_fp32_baseline_accepted():
    assert rc(p_r=448.0, v_r=448.0, expect_overflow=True, pv_accum="fp32", depth=1) == A.SA2PP_OK


def test_quant_sizes_follow_reference_tiling():
    prob = _problem(2, 30, 30, 17776, 64, causal=False)
    sz = A.QuantSizes()
    assert A.lib().sa2pp_quant_sizes(ctypes.byref(prob), ctypes.byref(sz)) == 0
    n_qt, n_kb = -(-17776 // 128), -(-17776 // 64)           # 139 query tiles, 278 key blocks
    assert (n_qt, n_kb) == (139, 278)
    assert sz.q_codes == 2 * 30 * n_qt * 128 * 64
    assert sz.k_codes == sz.v_codes == 2 * 30 * n_kb * 64 * 64
    assert sz.kv_meta == 2 * 30 * n_kb * (4 + 64) * 4


def test_config_mirror_matches_reference_rules():
    for p_r, v_r in sa.TABLE2_PAIRS:
        assert sa.RangeConfig(p_r, v_r, 2).product == 1008.0
    with pytest.raises(sa.RangeConfigError):
        sa.RangeConfig(448.0, 448.0, 1)
    with pytest.raises(sa.RangeConfigError, match=r"2016 > 1023\.5"):
        sa.RangeConfig(448.0, 4.5, 2)
    cfg = sa.AttentionConfig(seq_len=100, head_dim=64)
    assert cfg.scale == 0.125 and cfg.block_q == 128 and cfg.block_k == 64
    with pytest.raises(ValueError):
        sa.AttentionConfig(seq_len=100, head_dim=64, pv_accumulator="fp8")


def test_config_mirror_agrees_with_live_reference(lpattn):
    from lpattn.quantization import RangeConfig as RefRange, RangeConfigError as RefErr
    for args in [(224.0, 4.5, 2), (448.0, 4.5, 1), (448.0, 448.0, 1), (448.0, 4.5, 2), (112.0, 9.0, 2)]:
        ok_ref = ok_ours = True
        try:
            RefRange(*args)
        except RefErr:
            ok_ref = False
        try:
            sa.RangeConfig(*args)
        except sa.RangeConfigError:
            ok_ours = False
        assert ok_ref == ok_ours, args


def test_no_cpu_fallback():
    q = torch.zeros(1, 2, 64, 64)
    with pytest.raises(ValueError, match="CUDA"):
        sa.sageattn(q, q, q)


def test_reference_mirror_rejects_like_reference():
    import numpy as np
    z = np.zeros((1, 64, 48))
    with pytest.raises(ValueError):
        sa.attention_quantized(z, z, z, sa.AttentionConfig(seq_len=64, head_dim=48))
    with pytest.raises(ValueError):
        sa.attention_quantized(z, z, z[:, :32], sa.AttentionConfig(seq_len=64, head_dim=48))


def test_host_pipeline_validates_before_touching_the_gpu():
    """sa2pp_host_pipeline_create rejects bad problems/knobs with the reference's error classes
    before any CUDA call; run/destroy accept only real handles."""
    lib = A.lib()
    h = ctypes.c_void_p()
    prob = _problem(1, 4, 3, 128, 64, causal=False)  # heads_q % heads_kv != 0
    assert lib.sa2pp_host_pipeline_create(ctypes.byref(prob), A.SA2PP_BF16, 4, 2, ctypes.byref(h)) == A.SA2PP_ERR_INVALID
    prob = _problem(1, 4, 4, 128, 64, causal=False)
    assert lib.sa2pp_host_pipeline_create(ctypes.byref(prob), 7, 4, 2, ctypes.byref(h)) == A.SA2PP_ERR_INVALID
    assert lib.sa2pp_host_pipeline_create(ctypes.byref(prob), A.SA2PP_BF16, 0, 2, ctypes.byref(h)) == A.SA2PP_ERR_INVALID
    assert h.value is None
    assert lib.sa2pp_host_pipeline_run(None, None, None, None, None, None) == A.SA2PP_ERR_INVALID
    assert lib.sa2pp_host_pipeline_sync(None) == A.SA2PP_ERR_INVALID
    assert lib.sa2pp_host_pipeline_destroy(None) == A.SA2PP_OK


def test_conversion_halving_counters():
    """lpattn tests/test_attention.py:217-230 on the analytic RunReport counters the mirror reports:
    depth 1 converts every k=32 group sum, depth 2 every pair, MMA invocations are unchanged."""
    from paper_2505_21136_b200.api import _analytic_counts
    counts = {d: _analytic_counts(sa.AttentionConfig(seq_len=128, head_dim=32, range=sa.RangeConfig(224.0, 4.5, d)))
              for d in (1, 2)}
    assert counts[1][0] == 2 * counts[2][0]
    assert counts[1][1] == counts[2][1]


def test_integration_stub_is_valid_python_and_binds_declared_symbols():
    """The reference-side binding shown in INTEGRATION.md compiles and only names C entry points that
    include/sa2pp.h declares."""
    text = (ROOT / "INTEGRATION.md").read_text()
    block = re.search(r"```python\n(# lpattn/_b200\.py.*?)```", text, re.S).group(1)
    compile(block, "INTEGRATION.md", "exec")
    header = (ROOT / "include" / "sa2pp.h").read_text()
    called = set(re.findall(r"_lib\.(sa2pp_\w+)\(", block))
    called |= {f"sa2pp_host_pipeline_{f}" for f in re.findall(r'for _f in \(([^)]*)\)', block)[0].replace('"', "").replace(" ", "").split(",") if f}
    assert called and called <= set(declared_functions()), called - set(declared_functions())
    for name in re.findall(r"#.*?\b(sa2pp_[a-z_]+)\b", block):  # types named in comments exist too
        assert name in header, name


def test_analytic_counts_c_abi_equals_python_mirror():
    """sa2pp_analytic_counts (used by the host RunReport) equals the Python mirror of mma.py's
    counting on ragged, causal, depth-1/2 and FP32-accumulator configurations."""
    import ctypes
    from paper_2505_21136_b200.api import _analytic_counts, _problem
    for n, d, causal, depth, acc in ((100, 64, False, 2, "fp16"), (1000, 128, True, 1, "fp16"),
                                     (17776 // 8, 64, False, 2, "fp32"), (257, 128, True, 2, "fp16")):
        cfg = sa.AttentionConfig(seq_len=n, head_dim=d, num_heads=3, causal=causal, pv_accumulator=acc,
                                 range=sa.RangeConfig(224.0, 4.5, depth) if acc == "fp16"
                                 else sa.RangeConfig(448.0, 448.0, 1, expect_overflow=True))
        prob = _problem(1, 3, 3, n, d, causal=causal, pv_accum=acc, depth=cfg.range.buffering_depth,
                        p_r=cfg.range.p_r, v_r=cfg.range.v_r, expect_overflow=cfg.range.expect_overflow)
        conv, mma = ctypes.c_uint64(), ctypes.c_uint64()
        assert A.lib().sa2pp_analytic_counts(ctypes.byref(prob), ctypes.byref(conv), ctypes.byref(mma)) == A.SA2PP_OK
        assert (conv.value, mma.value) == _analytic_counts(cfg), (n, d, causal, depth, acc)


def test_sageattn_custom_op_fake_tensor_shapes():
    """torch.ops.sa2pp.sageattn propagates shapes and dtypes under FakeTensorMode (no GPU needed)."""
    import torch
    from torch._subclasses.fake_tensor import FakeTensorMode
    with FakeTensorMode():
        q = torch.empty(2, 300, 8, 64, dtype=torch.float16, device="cuda")
        k = torch.empty(2, 300, 2, 64, dtype=torch.float16, device="cuda")
        o = torch.ops.sa2pp.sageattn(q, k, k, "NHD", False, 0.125)
        assert o.shape == q.shape and o.dtype == q.dtype
