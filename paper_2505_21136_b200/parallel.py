"""Multi-GPU layouts for the path.

* Batch x head configs shard naturally: each rank owns a contiguous range of (batch, head)
  units (or of (batch, kv-head) groups under GQA) and runs sageattn on it.  There is no
  data-path collective; `shard_units` is the partition the bench uses.
* Long sequences use the Ulysses layout: every rank holds a sequence shard of all heads,
  one all-to-all turns that into full sequences of H/P heads, attention runs locally,
  and a second all-to-all restores the sequence sharding.  Smoothing statistics are
  per-head means over ALL tokens (quantization.py:133,147), so after the first exchange
  each rank's per-head computation is identical to the single-GPU one, and key blocks
  are still visited in ascending order (attention.py:6-8) -- results are bit-identical
  to one GPU.

The collectives are torch.distributed (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

from typing import Callable, Optional

import torch
import torch.distributed as dist


def shard_units(batch: int, heads: int, world: int, rank: int, group: int = 1) -> list[tuple[int, int]]:
    """(batch, head) units owned by `rank`: a contiguous, balanced slice of the B x H grid.

    With GQA (`group` query heads per KV head) units move in whole KV groups so every rank
    reads each K/V head it needs exactly once.
    """
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if heads % group:
        raise ValueError("heads must be a multiple of the GQA group")
    kv_units = batch * (heads // group)
    lo = kv_units * rank // world
    hi = kv_units * (rank + 1) // world
    out = []
    for u in range(lo, hi):
        b, g = divmod(u, heads // group)
        out.extend((b, g * group + i) for i in range(group))
    return out


def _a2a(x: torch.Tensor, group=None) -> torch.Tensor:
    out = torch.empty_like(x)
    dist.all_to_all_single(out, x.contiguous(), group=group)
    return out


def seq_to_head(x: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """[B, N/P, H, D] (sequence shard, all heads) -> [B, N, H/P, D] (all tokens, head shard)."""
    B, n, H, D = x.shape
    if H % world:
        raise ValueError(f"{H} heads do not split over {world} ranks")
    hp = H // world
    # chunk p of dim 0 goes to rank p: heads [p*hp, (p+1)*hp) of this rank's tokens
    send = x.reshape(B, n, world, hp, D).permute(2, 0, 1, 3, 4).contiguous()
    recv = _a2a(send, group)  # [P(source rank = token shard), B, n, hp, D]
    return recv.permute(1, 0, 2, 3, 4).reshape(B, world * n, hp, D)


def head_to_seq(x: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """Inverse of seq_to_head: [B, N, H/P, D] -> [B, N/P, H, D]."""
    B, N, hp, D = x.shape
    if N % world:
        raise ValueError(f"{N} tokens do not split over {world} ranks")
    n = N // world
    send = x.reshape(B, world, n, hp, D).permute(1, 0, 2, 3, 4).contiguous()
    recv = _a2a(send, group)  # [P(source rank = head shard), B, n, hp, D]
    return recv.permute(1, 2, 0, 3, 4).reshape(B, n, world * hp, D)


def ulysses_sageattn(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, is_causal: bool = False,
                     sm_scale: Optional[float] = None, *, group=None,
                     attn: Optional[Callable] = None, **kwargs) -> torch.Tensor:
    """Sequence-parallel sageattn (Ulysses).  q, k, v: this rank's [B, N/P, H, D] token shard.

    `attn(q, k, v, is_causal, sm_scale, **kwargs)` takes NHD full-sequence tensors; it defaults
    to the sm_100a sageattn (tests substitute a CPU oracle).
    """
    world = dist.get_world_size(group)
    if attn is None:
        from .api import sageattn

        def attn(q_, k_, v_, causal, scale, **kw):
            return sageattn(q_, k_, v_, "NHD", causal, scale, **kw)
    qh, kh, vh = (seq_to_head(t, world, group) for t in (q, k, v))
    oh = attn(qh, kh, vh, is_causal, sm_scale, **kwargs)
    return head_to_seq(oh, world, group)
