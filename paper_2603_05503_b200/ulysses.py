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
    """Closure running one head-sharded layer with ONE stacked exchange of Q, K and V
    (SURVEY 8.6): the send buffer interleaves the three tensors per token,
    [P_dst, B, N/P, 3, H/P, d], so a single all_to_all_single moves them and the receive buffer
    [P_src, B, N/P, 3, H/P, d] is, for batch 1, the token-ordered [1, N, 3, H/P, d]: Q, K and V
    are strided views of it (token stride 3 H/P d elements) that the kernel's TMA maps read
    directly, with no unpack copy.  The attention output [B, N, H/P, d] is, for batch 1, already
    the send layout [P_dst, N/P, H/P, d] of the return exchange.  `attention` maps [B, N, H/P, d]
    views (any token stride, head_dim contiguous) to a contiguous output of that shape (the
    rank's csa_sparse_attn_fwd).  Returns this rank's [B, N/P, H, d] output."""
    b, n_loc, h, d = q_loc.shape
    hp = h // world
    n = n_loc * world
    send = torch.empty((world, b, n_loc, 3, hp, d), dtype=q_loc.dtype, device=q_loc.device)
    recv = torch.empty_like(send)
    o_recv = torch.empty((world, b, n_loc, hp, d), dtype=q_loc.dtype, device=q_loc.device)

    def step():
        for s_, x in enumerate((q_loc, k_loc, v_loc)):
            send[:, :, :, s_].copy_(x.view(b, n_loc, world, hp, d).permute(2, 0, 1, 3, 4))
        dist.all_to_all_single(recv, send, group=group)
        if b == 1:
            qkv = recv.view(1, n, 3, hp, d)              # token order = source-rank order
        else:
            qkv = recv.permute(1, 0, 2, 3, 4, 5).reshape(b, n, 3, hp, d)
        o = attention(qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2])
        o_send = o.view(world, n_loc, hp, d) if b == 1 else \
            o.view(b, world, n_loc, hp, d).transpose(0, 1).contiguous()
        dist.all_to_all_single(o_recv.view(world, -1), o_send.reshape(world, -1), group=group)
        # [P_src = head group, B, N/P, H/P, d] -> [B, N/P, H, d]
        return o_recv.permute(1, 2, 0, 3, 4).reshape(b, n_loc, h, d)

    return step


def make_layer_step_chunked(q_loc, k_loc, v_loc, world: int, attention, chunks: int, group=None):
    """One head-sharded layer with the exchange overlapped with the attention: this
    rank's H/P heads are split into `chunks` head chunks; the stacked all-to-all of chunk c+1's
    Q, K, V (one all_to_all_single per chunk, layout as in make_layer_step) and the return
    exchange of chunk c-1's output run on a communication stream while chunk c's attention runs
    on the current stream.  attention(c, qh, kh, vh) maps chunk c's [B, N, H/(P chunks), d]
    views (heads c*hc .. of this rank) to a contiguous output of that shape.  Every rank must use
    the same `chunks`; the result equals make_layer_step's bit for bit (head-local attention, the
    same bytes moved).  On CPU tensors (gloo) the same schedule runs without streams."""
    b, n_loc, h, d = q_loc.shape
    hp = h // world
    if hp % chunks:
        raise ValueError(f"{hp} heads per rank not divisible into {chunks} chunks")
    hc = hp // chunks
    cuda = q_loc.is_cuda
    comm = torch.cuda.Stream(device=q_loc.device) if cuda else None
    n = n_loc * world
    kw = dict(dtype=q_loc.dtype, device=q_loc.device)
    # chunk c send: [P_dst, B, N/P, 3, hc, d] = heads p*hp + c*hc .. of this rank's tokens
    send = [torch.empty((world, b, n_loc, 3, hc, d), **kw) for _ in range(chunks)]
    recv = [torch.empty_like(x) for x in send]
    o_send = [torch.empty((world, b, n_loc, hc, d), **kw) for _ in range(chunks)]
    o_recv = [torch.empty_like(x) for x in o_send]
    out = torch.empty((b, n_loc, h, d), **kw)

    def ctx(stream):
        return torch.cuda.stream(stream) if cuda else _Null()

    def views(r):  # [P_src, B, N/P, 3, hc, d] -> Q, K, V [B, N, hc, d] (token order)
        qkv = r.view(1, n, 3, hc, d) if b == 1 else r.permute(1, 0, 2, 3, 4, 5).reshape(b, n, 3, hc, d)
        return qkv[:, :, 0], qkv[:, :, 1], qkv[:, :, 2]

    def step():
        cur = torch.cuda.current_stream(q_loc.device) if cuda else None
        ev_in, ev_out = [], []
        if cuda:
            comm.wait_stream(cur)  # inputs written on the current stream
        with ctx(comm):
            for c in range(chunks):
                for s_, x in enumerate((q_loc, k_loc, v_loc)):
                    send[c][:, :, :, s_].copy_(
                        x.view(b, n_loc, world, hp, d)[:, :, :, c * hc:(c + 1) * hc]
                        .permute(2, 0, 1, 3, 4))
                dist.all_to_all_single(recv[c], send[c], group=group)
                if cuda:
                    e = torch.cuda.Event()
                    e.record(comm)
                    ev_in.append(e)
        for c in range(chunks):
            if cuda:
                cur.wait_event(ev_in[c])
            oh = attention(c, *views(recv[c]))
            o_send[c].copy_(oh.view(b, world, n_loc, hc, d).permute(1, 0, 2, 3, 4))
            if cuda:
                e = torch.cuda.Event()
                e.record(cur)
                ev_out.append(e)
            with ctx(comm):
                if cuda:
                    comm.wait_event(ev_out[c])
                dist.all_to_all_single(o_recv[c], o_send[c], group=group)
                # [P_src = head group, B, N/P, hc, d] -> heads p*hp + c*hc .. of this rank's tokens
                out.view(b, n_loc, world, hp, d)[:, :, :, c * hc:(c + 1) * hc].copy_(
                    o_recv[c].permute(1, 2, 0, 3, 4))
        if cuda:
            cur.wait_stream(comm)
        return out

    return step


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
