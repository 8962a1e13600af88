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


class LayerExchange:
    """Buffers and views of one head-sharded layer exchange for `heads_per_chunk`
    of this rank's heads.  Send layout [P_dst, N/P, B, 3, hc, d]: Q, K, V of a token are
    interleaved and the batch (the CFG branches) sits inside the token, so ONE
    all_to_all_single moves all three and the receive buffer [P_src, N/P, B, 3, hc, d] IS the
    token-ordered [N, B, 3, hc, d]: qkv(s) is the strided [B, N, hc, d] view the kernel's TMA
    maps read in place (stride_b = 3 hc d, stride_n = 3 B hc d).  The attention writes its output
    straight into o_send [P_dst, N/P, B, hc, d] through the strided view out_view() (stride_b =
    hc d, stride_n = B hc d): the return exchange needs no pack either."""

    def __init__(self, b: int, n_loc: int, world: int, hc: int, d: int, dtype, device):
        self.b, self.n_loc, self.world, self.hc, self.d = b, n_loc, world, hc, d
        kw = dict(dtype=dtype, device=device)
        self.send = torch.empty((world, n_loc, b, 3, hc, d), **kw)
        self.recv = torch.empty_like(self.send)
        self.o_send = torch.empty((world, n_loc, b, hc, d), **kw)
        self.o_recv = torch.empty_like(self.o_send)

    def pack(self, xs, world: int, hp: int, h0: int) -> None:
        """send[p, t, b, s] = x_s[b, t, p hp + h0 : p hp + h0 + hc] for s = Q, K, V."""
        b, n_loc, hc, d = self.b, self.n_loc, self.hc, self.d
        for s_, x in enumerate(xs):
            self.send[:, :, :, s_].copy_(
                x.view(b, n_loc, world, hp, d)[:, :, :, h0:h0 + hc].permute(2, 1, 0, 3, 4))

    def qkv(self, s_: int) -> torch.Tensor:
        n = self.world * self.n_loc
        return self.recv.view(n, self.b, 3, self.hc, self.d)[:, :, s_].transpose(0, 1)

    def out_view(self) -> torch.Tensor:
        n = self.world * self.n_loc
        return self.o_send.view(n, self.b, self.hc, self.d).transpose(0, 1)

    def unpack(self, out: torch.Tensor, hp: int, h0: int) -> None:
        """o_recv [P_src = head group, N/P, B, hc, d] -> out[b, t, p hp + h0 ..] of this rank's
        token shard [B, N/P, H, d]."""
        b, n_loc, world, hc, d = self.b, self.n_loc, self.world, self.hc, self.d
        out.view(b, n_loc, world, hp, d)[:, :, :, h0:h0 + hc].copy_(
            self.o_recv.permute(2, 1, 0, 3, 4))


def make_layer_step(q_loc, k_loc, v_loc, world: int, attention, group=None, out=None):
    """Closure running one head-sharded layer: ONE stacked all-to-all of Q, K, V (LayerExchange),
    attention(q, k, v, out) on this rank's heads -- q, k, v and out are strided [B, N, H/P, d]
    views of the exchange buffers, read and written in place by the kernel (the rank's
    csa_sparse_attn_fwd) -- then the return all-to-all.  Returns this rank's [B, N/P, H, d]."""
    b, n_loc, h, d = q_loc.shape
    hp = h // world
    ex = LayerExchange(b, n_loc, world, hp, d, q_loc.dtype, q_loc.device)
    if out is None:
        out = torch.empty((b, n_loc, h, d), dtype=q_loc.dtype, device=q_loc.device)

    def step():
        ex.pack((q_loc, k_loc, v_loc), world, hp, 0)
        dist.all_to_all_single(ex.recv, ex.send, group=group)
        attention(ex.qkv(0), ex.qkv(1), ex.qkv(2), ex.out_view())
        dist.all_to_all_single(ex.o_recv, ex.o_send, group=group)
        ex.unpack(out, hp, 0)
        return out

    return step


def make_layer_step_chunked(q_loc, k_loc, v_loc, world: int, attention, chunks: int, group=None,
                            out=None, comm=None):
    """One head-sharded layer with the exchange overlapped with the attention: this
    rank's H/P heads are split into `chunks` head chunks, each with its own LayerExchange; the
    stacked all-to-all of chunk c+1 (and the return exchange of chunk c-1) runs on a
    communication stream while chunk c's attention runs on the current stream.
    attention(c, q, k, v, out) handles heads c*hc .. of this rank (strided views, written in
    place).  Every rank must use the same `chunks`; the result equals make_layer_step's bit for
    bit (head-local attention, the same bytes moved).  On CPU tensors (gloo) the same schedule
    runs without streams."""
    b, n_loc, h, d = q_loc.shape
    hp = h // world
    if hp % chunks:
        raise ValueError(f"{hp} heads per rank not divisible into {chunks} chunks")
    hc = hp // chunks
    cuda = q_loc.is_cuda
    if cuda and comm is None:
        comm = torch.cuda.Stream(device=q_loc.device)
    exs = [LayerExchange(b, n_loc, world, hc, d, q_loc.dtype, q_loc.device) for _ in range(chunks)]
    if out is None:
        out = torch.empty((b, n_loc, h, d), dtype=q_loc.dtype, device=q_loc.device)

    def ctx(stream):
        return torch.cuda.stream(stream) if cuda else _Null()

    def step():
        cur = torch.cuda.current_stream(q_loc.device) if cuda else None
        ev_in, ev_out = [], []
        if cuda:
            comm.wait_stream(cur)  # inputs written on the current stream
        with ctx(comm):
            for c, ex in enumerate(exs):
                ex.pack((q_loc, k_loc, v_loc), world, hp, c * hc)
                dist.all_to_all_single(ex.recv, ex.send, group=group)
                if cuda:
                    e = torch.cuda.Event()
                    e.record(comm)
                    ev_in.append(e)
        for c, ex in enumerate(exs):
            if cuda:
                cur.wait_event(ev_in[c])
            attention(c, ex.qkv(0), ex.qkv(1), ex.qkv(2), ex.out_view())
            if cuda:
                e = torch.cuda.Event()
                e.record(cur)
                ev_out.append(e)
            with ctx(comm):
                if cuda:
                    comm.wait_event(ev_out[c])
                dist.all_to_all_single(ex.o_recv, ex.o_send, group=group)
                ex.unpack(out, hp, c * hc)
        if cuda:
            cur.wait_stream(comm)
        return out

    return step


def make_layer_step_fused_out(q_loc, k_loc, v_loc, world: int, attention_scatter, group=None):
    """One head-sharded layer whose RETURN exchange is fused into the attention epilogue (SURVEY
    8.6 stretch): the output tensor [B, N/P, H, d] of every rank is a symmetric-memory buffer,
    and the kernel (csa_sparse_attn_fwd_scatter) stores each finished output row of token t
    straight into the buffer of the rank owning t's sequence shard, at this rank's head columns
    -- over NVLink peer mappings, as the tiles complete.  The Q/K/V exchange stays the stacked
    all_to_all_single of LayerExchange.  A device-side barrier of the symmetric buffers orders
    the peers' stores before the consumer's reads (and the previous layer's reads before the
    next stores).  attention_scatter(q, k, v, peer_ptrs, recv_like) runs this rank's heads.
    Returns step() -> this rank's [B, N/P, H, d] (the symmetric buffer itself)."""
    import torch.distributed._symmetric_memory as symm_mem

    b, n_loc, h, d = q_loc.shape
    hp = h // world
    grp = group if group is not None else dist.group.WORLD
    rank = dist.get_rank(grp)
    ex = LayerExchange(b, n_loc, world, hp, d, q_loc.dtype, q_loc.device)
    out = symm_mem.empty((b, n_loc, h, d), dtype=q_loc.dtype, device=q_loc.device)
    hdl = symm_mem.rendezvous(out, grp.group_name)
    esz = out.element_size()
    # this rank's first head inside every rank's receive buffer
    peer_ptrs = torch.tensor([int(hdl.buffer_ptrs[p]) + rank * hp * d * esz for p in range(world)],
                             dtype=torch.int64, device=q_loc.device)

    def step():
        ex.pack((q_loc, k_loc, v_loc), world, hp, 0)
        dist.all_to_all_single(ex.recv, ex.send, group=group)
        hdl.barrier(channel=0)   # every peer is done reading its previous output
        attention_scatter(ex.qkv(0), ex.qkv(1), ex.qkv(2), peer_ptrs, out)
        hdl.barrier(channel=1)   # every peer's rows have landed in this rank's buffer
        return out

    step.out = out  # the symmetric output buffer (this rank's [B, N/P, H, d])
    return step


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False
