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
