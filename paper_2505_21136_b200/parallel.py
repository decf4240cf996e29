"""Multi-GPU layouts for the path.

* Batch x head configs shard naturally with no data-path collective.  The unit of work is one
  128-row query tile of one (batch, head): `TilePlan` gives each rank a contiguous, balanced
  range of the flattened (b*H + h)*n_qt + tile space (balanced to one tile, e.g. CogVideoX's 60
  heads x 139 tiles over 8 ranks), runs the prepass for the heads (whole GQA groups) that range
  touches and the attention kernel on its tiles only (`sa2pp_attn_fwd_units`).  `shard_units` is
  the coarser whole-(batch, head) partition.
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

from dataclasses import dataclass
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


@dataclass(frozen=True)
class TilePlan:
    """Rank `rank`'s share of a (B, H, Hkv, N) problem in query-tile units.

    Units u = (b*H + h)*n_qt + t are split contiguously; the rank holds the flattened query
    heads [head_lo, head_hi) (extended to whole GQA groups, so kv heads
    [head_lo/group, head_hi/group) ) as a local problem of batch 1 and computes local units
    [unit_lo - head_lo*n_qt, unit_hi - head_lo*n_qt).  Flattening (b, h) is valid for HND
    inputs, where consecutive heads are a fixed stride apart across batch boundaries too.
    """

    batch: int
    heads: int
    kv_heads: int
    seq: int
    world: int
    rank: int

    @property
    def group(self) -> int:
        return self.heads // self.kv_heads

    @property
    def n_qt(self) -> int:
        return (self.seq + 127) // 128

    @property
    def total_units(self) -> int:
        return self.batch * self.heads * self.n_qt

    @property
    def unit_lo(self) -> int:
        return self.total_units * self.rank // self.world

    @property
    def unit_hi(self) -> int:
        return self.total_units * (self.rank + 1) // self.world

    @property
    def head_lo(self) -> int:
        h = self.unit_lo // self.n_qt
        return h - h % self.group

    @property
    def head_hi(self) -> int:
        if self.unit_hi == self.unit_lo:
            return self.head_lo
        h = (self.unit_hi - 1) // self.n_qt + 1
        return -(-h // self.group) * self.group

    @property
    def local_heads(self) -> int:
        return self.head_hi - self.head_lo

    @property
    def local_units(self) -> tuple[int, int]:
        base = self.head_lo * self.n_qt
        return self.unit_lo - base, self.unit_hi - base

    def unit_rows(self, u: int) -> tuple[int, int, int]:
        """(flattened head, first row, end row) of global unit u."""
        h, t = divmod(u, self.n_qt)
        return h, t * 128, min(self.seq, t * 128 + 128)


def tile_plan(batch: int, heads: int, kv_heads: int, seq: int, world: int, rank: int) -> TilePlan:
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    if heads % kv_heads:
        raise ValueError("heads must be a multiple of kv_heads")
    return TilePlan(batch, heads, kv_heads, seq, world, rank)


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
