"""The exactness certificate behind the parallel channel means (csrc/prepass.cu means_finalize).

numpy's x.mean(axis=0) is a sequential float64 sum (quantization.py:133,147).  The GPU path sums
512-row chunks in parallel and accepts the result only when N * max|x| < 2^53 * u, u the ulp of the
channel's smallest nonzero element in the input format.  Under that condition every partial sum is
a multiple of u below 2^53 * u, so it is representable and no addition rounds: the sequential sum,
any chunked sum and the exact sum agree.  Checked here on bf16/fp16-representable data with numpy
and exact integer arithmetic; the GPU side is tests/test_gpu_parity.py::
test_parallel_certified_means_match_numpy.
"""

from fractions import Fraction

import numpy as np
import pytest

FORMATS = {"bf16": (7, 127), "fp16": (10, 15)}  # mantissa bits, exponent bias


def to_format(x, fmt):
    if fmt == "fp16":
        return x.astype(np.float16).astype(np.float64)
    b = x.astype(np.float32).view(np.uint32)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000  # round to nearest even bf16
    return b.view(np.float32).astype(np.float64)


def certificate(col, fmt):
    mb, bias = FORMATS[fmt]
    nz = np.abs(col[col != 0])
    if nz.size == 0:
        return True
    e_min = max(int(np.floor(np.log2(nz.min()))) + bias, 1)  # biased; subnormals share e = 1
    ulp_exp = e_min - bias - mb
    return len(col) * nz.max() < 2.0 ** (53 + ulp_exp)


def exact_sum(col, fmt):
    mb, bias = FORMATS[fmt]
    u_exp = 1 - bias - mb  # smallest ulp of the format: every element is an integer multiple of it
    ints = [int(v * 2.0 ** -u_exp) for v in col]
    assert all(Fraction(i, 2 ** -u_exp) == Fraction(v) for i, v in zip(ints, col))
    return Fraction(sum(ints), 2 ** -u_exp)


@pytest.mark.parametrize("fmt", ["bf16", "fp16"])
@pytest.mark.parametrize("spread", [0.0, 1.0, 3.0, 8.0])
def test_certified_sums_are_exact_in_any_order(fmt, spread):
    rng = np.random.default_rng(int(spread * 10) + len(fmt))
    n = 4096
    for trial in range(6):
        col = rng.standard_normal(n) * np.exp(rng.standard_normal(n) * spread)
        if fmt == "fp16":
            col = np.clip(col, -6e4, 6e4)
        col = to_format(col, fmt)
        seq = 0.0
        for v in col:  # numpy's order for mean(axis=0) over rows
            seq += v
        chunks = [col[i:i + 512] for i in range(0, n, 512)]
        chunked = 0.0
        for c in reversed(chunks):  # a different order: chunk sums added last-first
            s = 0.0
            for v in c:
                s += v
            chunked += s
        exact = exact_sum(col, fmt)
        if spread == 0.0:
            assert certificate(col, fmt)  # N(0,1) data: the common case the parallel path relies on
        if certificate(col, fmt):
            assert Fraction(seq) == Fraction(chunked) == exact, (fmt, spread, trial)
        else:
            assert spread > 0.0  # only a wide exponent spread can fail it


def test_certificate_fails_where_rounding_happens():
    """A value far below the others' ulp: the sequential sum rounds, the certificate must refuse."""
    col = to_format(np.array([1.0] * 1000 + [2.0 ** -60] + [1.0] * 1000), "bf16")
    assert not certificate(col, "bf16")
    seq = 0.0
    for v in col:
        seq += v
    assert Fraction(seq) != exact_sum(col, "bf16")
