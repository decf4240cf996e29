"""Multi-process (gloo, world size 2) coverage of the N>1 host logic on CPU.

* batch x head sharding: every (b, h) unit owned by exactly one rank, GQA groups kept whole;
* Ulysses all-to-all layout: sequence shards -> head shards -> attention -> sequence shards
  is identical to running the reference pipeline on the full sequence (the oracle stands in
  for the GPU kernel here; per-head computation is unchanged by the exchange).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2505_21136_b200.parallel import head_to_seq, seq_to_head, shard_units, ulysses_sageattn


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("B,H,group,world", [(4, 32, 1, 8), (2, 30, 1, 8), (8, 32, 4, 8), (1, 32, 1, 2), (3, 5, 1, 4)])
def test_shard_units_partition(B, H, group, world):
    seen = []
    for r in range(world):
        units = shard_units(B, H, world, r, group)
        # GQA groups stay together
        for i in range(0, len(units), group):
            b, h = units[i]
            assert h % group == 0 and units[i: i + group] == [(b, h + k) for k in range(group)]
        seen += units
    assert sorted(seen) == [(b, h) for b in range(B) for h in range(H)]
    sizes = [len(shard_units(B, H, world, r, group)) for r in range(world)]
    assert max(sizes) - min(sizes) <= group


def _oracle_attn(q, k, v, causal, scale):
    """NHD [B, N, h, D] torch -> NHD output via the CPU oracle, head by head."""
    from oracle import sage_cpu as oc
    B, N, h, D = q.shape
    out = np.empty((B, N, h, D))
    for b in range(B):
        for hh in range(h):
            cfg = oc.AttentionConfig(seq_len=N, head_dim=D, causal=causal, softmax_scale=scale)
            out[b, :, hh] = oc.attention_quantized(q[b, :, hh].numpy(), k[b, :, hh].numpy(),
                                                   v[b, :, hh].numpy(), cfg).output
    return torch.from_numpy(out)


def _worker(rank, world, port, causal):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(7)
        B, N, H, D = 1, 256, 4, 64
        q, k, v = (torch.randn(B, N, H, D, generator=g, dtype=torch.float64) for _ in range(3))
        n = N // world
        sl = slice(rank * n, (rank + 1) * n)
        # layout round trip is exact
        x = q[:, sl]
        assert torch.equal(head_to_seq(seq_to_head(x, world), world), x)
        # head shard after the exchange holds all tokens of this rank's heads
        hp = H // world
        assert torch.equal(seq_to_head(x, world), q[:, :, rank * hp:(rank + 1) * hp])
        out = ulysses_sageattn(q[:, sl], k[:, sl], v[:, sl], causal, None, attn=_oracle_attn)
        full = _oracle_attn(q, k, v, causal, None)
        assert torch.equal(out, full[:, sl])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("causal", [False, True])
def test_ulysses_gloo_world2_matches_single_process(causal):
    mp.spawn(_worker, args=(2, _free_port(), causal), nprocs=2, join=True)


# ----------------------------------------------------------------------------- query-tile sharding
from paper_2505_21136_b200.parallel import tile_plan  # noqa: E402


@pytest.mark.parametrize("B,H,Hkv,N,world", [(2, 30, 30, 17776, 8), (8, 32, 8, 8192, 8), (4, 32, 32, 16384, 3),
                                              (1, 4, 2, 300, 2), (1, 2, 2, 100, 4)])
def test_tile_plan_partition(B, H, Hkv, N, world):
    """Every query tile of every (b, h) belongs to exactly one rank, ranks differ by at most one tile,
    and each rank's local problem (whole GQA groups) contains its tiles."""
    seen = []
    sizes = []
    for r in range(world):
        p = tile_plan(B, H, Hkv, N, world, r)
        lo, hi = p.local_units
        assert 0 <= lo <= hi <= p.local_heads * p.n_qt
        assert p.head_lo % p.group == 0 and p.head_hi % p.group == 0
        assert p.head_lo * p.n_qt <= p.unit_lo and p.unit_hi <= p.head_hi * p.n_qt
        seen += range(p.unit_lo, p.unit_hi)
        sizes.append(p.unit_hi - p.unit_lo)
    assert seen == list(range(B * H * ((N + 127) // 128)))
    assert max(sizes) - min(sizes) <= 1


def _tile_worker(rank, world, port, causal, group):
    """The bench's sharded path with the oracle standing in for the kernel: each rank takes its
    TilePlan, quantizes/attends its local heads (HND, batch flattened into heads, as bench.py
    does) and keeps only its query tiles; the gathered tiles equal the single-process result."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sage_cpu as oc
        g = torch.Generator().manual_seed(11)
        B, H, N, D = 2, 2 * group, 300, 64
        Hkv = H // group
        q = torch.randn(B, H, N, D, generator=g, dtype=torch.float64)
        k = torch.randn(B, Hkv, N, D, generator=g, dtype=torch.float64)
        v = torch.randn(B, Hkv, N, D, generator=g, dtype=torch.float64)
        cfg = oc.AttentionConfig(seq_len=N, head_dim=D, causal=causal)

        def head_out(qf, kf, vf, hq):  # flattened HND heads, GQA: kv head hq // group
            return oc.attention_quantized(qf[hq].numpy(), kf[hq // group].numpy(), vf[hq // group].numpy(), cfg).output

        p = tile_plan(B, H, Hkv, N, world, rank)
        qf, kf, vf = q.reshape(B * H, N, D), k.reshape(B * Hkv, N, D), v.reshape(B * Hkv, N, D)
        # local problem: flattened heads [head_lo, head_hi), kv heads [head_lo/group, head_hi/group)
        ql = qf[p.head_lo:p.head_hi]
        kl, vl = kf[p.head_lo // group:p.head_hi // group], vf[p.head_lo // group:p.head_hi // group]
        lo, hi = p.local_units
        mine = {}
        for lu in range(lo, hi):
            hl, t = divmod(lu, p.n_qt)
            o = head_out(ql, kl, vl, hl)
            mine[p.head_lo * p.n_qt + lu] = torch.from_numpy(o[t * 128:min(N, t * 128 + 128)])
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        allu = {}
        for d in gathered:
            assert not set(d) & set(allu)
            allu.update(d)
        assert sorted(allu) == list(range(p.total_units))
        for u, o in allu.items():
            hq, r0, r1 = p.unit_rows(u)
            ref = head_out(qf, kf, vf, hq)[r0:r1]
            assert torch.equal(o, torch.from_numpy(ref))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("causal,group", [(False, 1), (True, 2)])
def test_tile_shard_gloo_world2_matches_single_process(causal, group):
    mp.spawn(_tile_worker, args=(2, _free_port(), causal, group), nprocs=2, join=True)
