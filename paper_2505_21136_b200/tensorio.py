"""The reference's on-disk tensor container (LPATTN-TENSOR v1, tensorio.py:1-114), for exchanging
inputs and outputs byte-for-byte between the CPU reference and the B200 path.

Layout (little-endian): 16-byte magic ``LPATTN-TENSOR\\0\\0\\0``, u64 version (1), u64 rank, rank x u64
dims, row-major float32 payload; optional JSON sidecar ``<file>.meta.json``.  `load` returns the
tensor on a device (through pinned host memory), `save` writes one from any device.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import torch

MAGIC = b"LPATTN-TENSOR\x00\x00\x00"
VERSION = 1


class TensorFormatError(ValueError):
    """Not a valid LPATTN-TENSOR v1 file (same name and base class as the reference's)."""


def _sidecar(path: Path) -> Path:
    return path.with_suffix(path.suffix + ".meta.json")


def write_tensor(path, array, meta: dict | None = None) -> None:
    arr = np.ascontiguousarray(np.asarray(array), dtype="<f4")
    header = np.array([VERSION, arr.ndim, *arr.shape], dtype="<u8")
    path = Path(path)
    path.write_bytes(MAGIC + header.tobytes() + arr.tobytes())
    if meta is not None:
        _sidecar(path).write_text(json.dumps(meta, indent=2, sort_keys=True) + "\n")


def read_tensor(path) -> np.ndarray:
    raw = Path(path).read_bytes()
    if raw[:16] != MAGIC:
        raise TensorFormatError(f"{path}: bad magic {raw[:16]!r}")
    if len(raw) < 32:
        raise TensorFormatError(f"{path}: truncated header")
    version, rank = np.frombuffer(raw, dtype="<u8", count=2, offset=16)
    if int(version) != VERSION:
        raise TensorFormatError(f"{path}: unsupported version {int(version)}")
    rank = int(rank)
    off = 32 + 8 * rank
    if len(raw) < off:
        raise TensorFormatError(f"{path}: truncated header")
    shape = tuple(int(s) for s in np.frombuffer(raw, dtype="<u8", count=rank, offset=32))
    count = int(np.prod(shape, dtype=np.int64)) if rank else 1
    nbytes = len(raw) - off
    if nbytes < 4 * count:
        raise TensorFormatError(f"{path}: truncated payload")
    if nbytes > 4 * count:
        raise TensorFormatError(f"{path}: trailing bytes")
    return np.frombuffer(raw, dtype="<f4", count=count, offset=off).reshape(shape).astype(np.float32)


def load(path, device="cuda", dtype=torch.float32) -> torch.Tensor:
    """Read a tensor file straight onto `device` (pinned staging, non-blocking copy)."""
    host = torch.from_numpy(read_tensor(path))
    if torch.device(device).type == "cuda":
        host = host.pin_memory()
    return host.to(device=device, dtype=dtype, non_blocking=True)


def save(path, tensor: torch.Tensor, meta: dict | None = None) -> None:
    write_tensor(path, tensor.detach().to("cpu", torch.float32).numpy(), meta)
