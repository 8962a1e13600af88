"""Multi-process (world size 2, gloo, CPU) tests of the head-sharded exchange used by the
multi-GPU path: sequence-sharded -> head-sharded -> back is the identity, each rank receives
exactly its heads' full-sequence tensors, and a head-local operation commutes with the exchange
(so per-head results cannot depend on the number of ranks)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_05503_b200 import ulysses


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, batch, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(3)
        n, h, d = 12, 4, 8
        x = torch.randn((batch, n, h, d), generator=g)       # identical on every rank
        x_loc = ulysses.sequence_shard(x, world, rank)
        xh = ulysses.scatter_heads(x_loc, world)
        h0, h1 = ulysses.head_range(h, world, rank)
        ok_scatter = torch.equal(xh, x[:, :, h0:h1])
        back = ulysses.gather_heads(xh, world)
        ok_roundtrip = torch.equal(back, x_loc)
        # a head-local op (per-head scaling by the head index) commutes with the exchange
        scale = torch.arange(h0, h1, dtype=x.dtype).view(1, 1, -1, 1) + 1
        seen = {}

        def attn(q, k, v):  # the stacked exchange hands the kernel strided views (no unpack)
            seen["stride"] = q.stride()
            seen["qkv"] = (torch.equal(q, x[:, :, h0:h1]) and torch.equal(k, x[:, :, h0:h1])
                           and torch.equal(v, x[:, :, h0:h1]))
            return q * scale

        step = ulysses.make_layer_step(x_loc, x_loc, x_loc, world, attn)
        y_loc = step()
        hp_ = h1 - h0
        ok_views = seen["qkv"] and (batch > 1 or seen["stride"][1] == 3 * hp_ * d)
        ref = (x * (torch.arange(h, dtype=x.dtype).view(1, 1, -1, 1) + 1))
        ok_layer = torch.equal(y_loc, ulysses.sequence_shard(ref, world, rank))
        # a balanced head order (folded into the projections in a model): rank r receives the
        # heads perm[r*H/P:(r+1)*H/P] and the layer still commutes with the exchange
        perm = ulysses.balance_heads([5.0, 1.0, 4.0, 2.0], world)
        xp = x[:, :, perm]
        xph = ulysses.scatter_heads(ulysses.sequence_shard(xp, world, rank), world)
        ok_perm = torch.equal(xph, x[:, :, perm[h0:h1]])
        # head-chunked overlapped schedule: identical result for every chunk count
        ok_chunk = True
        for chunks in (1, 2):
            stepc = ulysses.make_layer_step_chunked(
                x_loc, x_loc, x_loc, world,
                lambda c, q, k, v, hc=(h1 - h0) // chunks: q * (scale[:, :, c * hc:(c + 1) * hc]),
                chunks)
            ok_chunk &= torch.equal(stepc(), y_loc)
        results[rank] = (ok_scatter, ok_roundtrip, ok_layer and ok_perm and ok_chunk and ok_views)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("batch", [1, 2])
def test_ulysses_exchange_gloo_world2(batch):
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), batch, results), nprocs=2, join=True)
    assert dict(results) == {0: (True, True, True), 1: (True, True, True)}


def test_balance_heads_lpt():
    cost = [9, 1, 8, 2, 7, 3, 6, 4]
    for world in (1, 2, 4, 8):
        perm = ulysses.balance_heads(cost, world)
        assert sorted(perm) == list(range(8))
        hp = 8 // world
        loads = [sum(cost[h] for h in perm[r * hp:(r + 1) * hp]) for r in range(world)]
        assert max(loads) - min(loads) <= max(cost)  # LPT: spread within one job
    assert ulysses.balance_heads(cost, 2) == [0, 1, 6, 7, 2, 3, 4, 5]  # 20 / 20
    with pytest.raises(ValueError):
        ulysses.balance_heads(cost, 3)


def test_head_range_and_shard_checks():
    assert ulysses.head_range(40, 8, 3) == (15, 20)
    with pytest.raises(ValueError):
        ulysses.head_range(40, 3, 0)
    with pytest.raises(ValueError):
        ulysses.sequence_shard(torch.zeros(1, 10, 2, 2), 3, 0)
