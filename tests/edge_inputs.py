"""Adversarial prepass inputs shared by the CPU (oracle vs live reference) and GPU (kernel vs oracle)
tests: exact rounding ties, huge channel offsets, zeros and FP32 subnormals."""

import numpy as np


def exact_ties():
    """amax 127 -> scale 1: codes are RNE of half-integers; V colmax 4.5 -> scale 1, E4M3 ties."""
    rng = np.random.default_rng(11)
    n, d = 256, 64
    q = (rng.integers(-254, 255, size=(2, n, d)) / 2.0).astype(np.float32)
    q[:, ::128, :] = 127.0  # pin amax of every 128-row tile
    k = q[:, ::-1, :].copy()
    k[:, ::64, :] = -127.0  # every 64-row block
    ties = np.array([1.0625, 1.1875, 0.0009765625, 0.0029296875, 2.25 + 0.125, 3.5 + 0.25, -1.0625, 0.0],
                    dtype=np.float32)
    v = ties[rng.integers(0, len(ties), size=(2, n, d))].astype(np.float32)
    v[:, ::64, :] = 4.5
    return q, k, v, False


def huge_offsets():
    """|mean| ~ 1e6 x the spread: the FP32 fast path is not exact, the FP64 one must run."""
    rng = np.random.default_rng(12)
    n, d = 200, 128
    base = rng.normal(size=(1, 1, d)) * 1e4
    q = (base + rng.normal(size=(2, n, d)) * 1e-2).astype(np.float32)
    k = (base[:, :, ::-1] + rng.normal(size=(2, n, d)) * 1e-2).astype(np.float32)
    v = rng.normal(size=(2, n, d)).astype(np.float32)
    return q, k, v, True


def zeros_subnormals():
    rng = np.random.default_rng(13)
    n, d = 300, 64
    q = rng.normal(size=(2, n, d)).astype(np.float32)
    k = rng.normal(size=(2, n, d)).astype(np.float32)
    v = rng.normal(size=(2, n, d)).astype(np.float32)
    q[0, 5:40] = 0.0
    k[1, 70:90] = 0.0
    v[0, :, 3] = 0.0
    v[1, 10:20, :] = np.float32(1e-40)
    k[0, 100:110, :] = np.float32(-3e-39)
    v[1, 128:192, 7] = np.float32(4.5) * np.array([1.0, 1.0625, 0.5, 0.03125, 0.0009765625] * 12 + [1.0] * 4,
                                                   dtype=np.float32)
    return q, k, v, True


def tiny_blocks():
    """Whole blocks / block channels whose amax is below 2^-100 (subnormals mixed with zeros): the f32
    reciprocal of the scale would overflow, so the exact FP64 path must run."""
    rng = np.random.default_rng(14)
    n, d = 256, 64
    q = rng.normal(size=(2, n, d)).astype(np.float32)
    k = rng.normal(size=(2, n, d)).astype(np.float32)
    v = rng.normal(size=(2, n, d)).astype(np.float32)
    v[0, 64:128, 5] = (np.float32(1e-40) * rng.integers(0, 3, size=64)).astype(np.float32)  # subnormal + zeros
    v[1, 128:192, 9] = np.float32(3e-38) * rng.choice([-1.0, 0.0, 0.5, 1.0], size=64).astype(np.float32)
    v[1, 192:256, :] = np.float32(2e-39) * rng.integers(-2, 3, size=(64, d)).astype(np.float32)  # a whole block
    k[1, 0:64, :] = (np.float32(1e-39) * rng.integers(-3, 4, size=(64, d))).astype(np.float32)  # K block amax tiny
    q[0, 0:128, :] = (np.float32(5e-39) * rng.normal(size=(128, d))).astype(np.float32)  # Q tile amax tiny
    return q, k, v, False


CASES = {"exact_ties": exact_ties, "huge_offsets": huge_offsets, "zeros_subnormals": zeros_subnormals,
         "tiny_blocks": tiny_blocks}
