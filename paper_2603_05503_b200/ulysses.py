"""Head-sharded multi-GPU attention layer: the Ulysses all-to-all exchange (plumbing).

Heads are independent and every plan cell belongs to one head, so a
layer is partitioned by head over the P ranks of the process group.  Activations arrive
sequence-sharded ([batch, N/P, H, d] per rank); one all-to-all turns them into head-sharded
full-sequence tensors ([batch, N, H/P, d]) for the rank's heads, the calibrated sparse attention
runs on those heads (csa_sparse_attn_fwd, plan cells of the rank's heads only), and a second
all-to-all returns the output to the sequence-sharded layout.  The exchange is plain
torch.distributed (NCCL on GPUs, gloo in the CPU tests); every arithmetic step is in libcsa.so.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def head_range(n_heads: int, world: int, rank: int) -> tuple[int, int]:
    if n_heads % world:
        raise ValueError(f"{n_heads} heads not divisible by {world} ranks")
    hp = n_heads // world
    return rank * hp, (rank + 1) * hp


def balance_heads(cost, world: int) -> list[int]:
    """Head order for the exchange (SURVEY 8.6 load balance): heads differ in kept area, a rank's
    time is the sum over its heads, so assign heads longest-first to the least-loaded rank that
    still has room (every rank takes H/P heads: the all-to-all splits stay equal); ties -> lower
    rank.  Returns perm (position -> head), rank r's heads at perm[r*H/P:(r+1)*H/P] ascending.
    A model folds perm into its QKV projection rows and the inverse into its output projection,
    so the reordering costs nothing at run time; the exchange itself is unchanged."""
    n = len(cost)
    if n % world:
        raise ValueError(f"{n} heads not divisible by {world} ranks")
    hp = n // world
    load, groups = [0.0] * world, [[] for _ in range(world)]
    for h in sorted(range(n), key=lambda x: (-float(cost[x]), x)):
        r = min((r for r in range(world) if len(groups[r]) < hp), key=lambda r: (load[r], r))
        groups[r].append(h)
        load[r] += float(cost[h])
    return [h for g in groups for h in sorted(g)]


def scatter_heads(x_loc: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """[B, N/P, H, d] (this rank's tokens, all heads) -> [B, N, H/P, d] (all tokens, this rank's
    heads).  Send block p holds head group p; the received blocks are in source-rank order, i.e.
    in token order."""
    b, n_loc, h, d = x_loc.shape
    hp = h // world
    send = x_loc.view(b, n_loc, world, hp, d).permute(2, 0, 1, 3, 4).contiguous()
    recv = torch.empty_like(send)                    # [P_src, B, N/P, H/P, d]
    dist.all_to_all_single(recv, send, group=group)
    if b == 1:
        return recv.view(1, world * n_loc, hp, d)    # already token-ordered
    return recv.permute(1, 0, 2, 3, 4).reshape(b, world * n_loc, hp, d)


def gather_heads(o_head: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """[B, N, H/P, d] (all tokens, this rank's heads) -> [B, N/P, H, d] (this rank's tokens,
    all heads).  Inverse of scatter_heads."""
    b, n, hp, d = o_head.shape
    n_loc = n // world
    send = o_head.view(b, world, n_loc, hp, d).permute(1, 0, 2, 3, 4).contiguous()
    recv = torch.empty_like(send)                    # [P_src (head group), B, N/P, H/P, d]
    dist.all_to_all_single(recv, send, group=group)
    return recv.permute(1, 2, 0, 3, 4).reshape(b, n_loc, world * hp, d)


def sequence_shard(x: torch.Tensor, world: int, rank: int) -> torch.Tensor:
    """This rank's contiguous token shard of a [B, N, H, d] tensor (N divisible by P)."""
    n = x.shape[1]
    if n % world:
        raise ValueError(f"{n} tokens not divisible by {world} ranks")
    s = n // world
    return x[:, rank * s:(rank + 1) * s].contiguous()


def make_layer_step(q_loc, k_loc, v_loc, world: int, attention, group=None):
    """Closure running one head-sharded layer: scatter Q, K, V -> attention(q, k, v) on this
    rank's heads -> gather O.  `attention` maps [B, N, H/P, d] tensors to an output of the same
    shape (the rank's csa_sparse_attn_fwd)."""

    def step():
        qh = scatter_heads(q_loc, world, group)
        kh = scatter_heads(k_loc, world, group)
        vh = scatter_heads(v_loc, world, group)
        return gather_heads(attention(qh, kh, vh), world, group)

    return step
