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

        def attn(q, k, v, out):  # strided views of the exchange buffers, written in place
            seen["stride"] = (q.stride(), out.stride())
            seen["qkv"] = (torch.equal(q, x[:, :, h0:h1]) and torch.equal(k, x[:, :, h0:h1])
                           and torch.equal(v, x[:, :, h0:h1]))
            out.copy_(q * scale)

        step = ulysses.make_layer_step(x_loc, x_loc, x_loc, world, attn)
        y_loc = step()
        hp_ = h1 - h0
        ok_views = seen["qkv"] and seen["stride"] == (
            (3 * hp_ * d, 3 * batch * hp_ * d, d, 1), (hp_ * d, batch * hp_ * d, d, 1))
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
                lambda c, q, k, v, out, hc=(h1 - h0) // chunks:
                    out.copy_(q * scale[:, :, c * hc:(c + 1) * hc]),
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


def _denoise_worker(rank, world, port, chunks, results):
    """CPU rehearsal of pipeline.ShardedDenoiseStep: T x L layers, CFG batch 2, head-chunked
    stacked exchange, with the fp64 oracle standing in for the kernel on each rank's heads."""
    import numpy as np

    import oracle
    from paper_2603_05503_b200 import inputs, pipeline

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lay = inputs.Layout(2, 5, 25, 64)               # N = 250, ragged last block
        T, L, H, B, d, S = 2, 2, 4, 2, 64, 2
        scale = 1.0 / np.sqrt(d)
        rng = np.random.default_rng(0)                  # identical on every rank
        masks = (rng.random((T, L, H, lay.NB, lay.NB)) < 0.5).astype(np.uint8)
        masks[..., np.arange(lay.NB), np.arange(lay.NB)] = 1
        perm = ulysses.balance_heads([3.0, 1.0, 2.0, 4.0], world)
        hp = H // world
        mine = perm[rank * hp:(rank + 1) * hp]
        full = [inputs.qkv(B, lay.N, H, d, seed=10 + s) for s in range(S)]   # [B, N, H, d]
        loc = [[ulysses.sequence_shard(x[:, :, perm].float(), world, rank) for x in f]
               for f in full]
        o = [torch.zeros_like(loc[s][0]) for s in range(S)]

        def oracle_attention(t, l, c, qh, kh, vh, out):
            hc = qh.shape[2]
            for b in range(B):
                for j in range(hc):
                    h = mine[c * hc + j]
                    r, _ = oracle.masked_attention_rows(qh[b, :, j].double().numpy(),
                                                        kh[b, :, j].double().numpy(),
                                                        vh[b, :, j].double().numpy(), scale,
                                                        lay.B, masks[t, l, h])
                    out[b, :, j] = torch.from_numpy(r).float()

        step = pipeline.ShardedDenoiseStep(None, world, [x[0] for x in loc], [x[1] for x in loc],
                                           [x[2] for x in loc], o, chunks=chunks,
                                           attention=oracle_attention, T=T, L=L)
        ok = True
        n_loc = lay.N // world
        for t in range(T):
            step.run(t)
            l = L - 1                                   # the last layer written to o[l % S]
            q, k, v = full[l % S]
            for p_, h in enumerate(perm):
                for b in range(B):
                    ref, _ = oracle.masked_attention_rows(q[b, :, h].double().numpy(),
                                                          k[b, :, h].double().numpy(),
                                                          v[b, :, h].double().numpy(), scale,
                                                          lay.B, masks[t, l, h])
                    got = o[l % S][b, :, p_].double().numpy()
                    ok &= bool(np.abs(got - ref[rank * n_loc:(rank + 1) * n_loc]).max() < 1e-6)
        results[rank] = ok
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("chunks", [1, 2])
def test_sharded_denoise_step_schedule_gloo_world2(chunks):
    """f4 on N ranks, rehearsed on CPU: the sharded denoising step's exchange / chunk / layer
    schedule delivers every rank's token shard of every head's masked attention (the oracle in
    place of the kernel), for the CFG batch and the LPT head order."""
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_denoise_worker, args=(2, _free_port(), chunks, results), nprocs=2, join=True)
    assert dict(results) == {0: True, 1: True}
