"""`torch.ops.sa2pp.sageattn`: the north-star drop-in registered as a PyTorch custom operator.

The operator has the reference signature `sageattn(q, k, v, tensor_layout, is_causal, sm_scale)`
and a fake (meta) implementation, so it composes with FakeTensor shape propagation, torch.compile
graphs (as an opaque call into the sm_100a library) and `torch.library.opcheck`.  Its real
implementation is `api.sageattn` on the caller's current stream: the C-ABI library does all the
arithmetic, there is no CPU kernel.
"""

from __future__ import annotations

from typing import Optional

import torch

from . import api


@torch.library.custom_op("sa2pp::sageattn", mutates_args=(), device_types="cuda")
def sageattn_op(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, tensor_layout: str = "HND",
                is_causal: bool = False, sm_scale: Optional[float] = None) -> torch.Tensor:
    return api.sageattn(q, k, v, tensor_layout, is_causal, sm_scale)


@sageattn_op.register_fake
def _(q, k, v, tensor_layout="HND", is_causal=False, sm_scale=None):
    if tensor_layout not in ("HND", "NHD"):
        raise ValueError(f"tensor_layout must be 'HND' or 'NHD', got {tensor_layout!r}")
    if q.dim() != 4 or k.dim() != 4 or v.dim() != 4:
        raise ValueError("q, k, v must be 4-D")
    if not (q.dtype == k.dtype == v.dtype):
        raise ValueError("q, k, v must share one dtype")
    return torch.empty_like(q)
