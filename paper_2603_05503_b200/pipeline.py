"""Whole-schedule runtime (f4): the calibrated plan dictionary over every (t, l, h) cell and the
attention of one denoising step over all layers, CFG batch 2, replayed as a CUDA graph.

PAPER.md:
  * the dictionary: calibration over |D| prompts for every timestep t, layer l and head h
    (P:532-571), repetitive heads from the spatial-similarity statistic, and the
    timestep-dependent threshold eps(t) of Eq. eq:epsilon_schedule with the paper's
    fitted constants: high-step A(N) = 0.796 + 1.41e-6 N, C = 0.99, k = 16 or the
    4-step distilled (LightX2V) A = 0.763, C = 0.863, k = 5.64;
  * CFG: masks and similarity are calibrated on the conditional branch only, and the same cell
    plan serves both branches at inference -- here batch 2 of one launch;
  * a denoising step runs the sparse attention of every layer with the cell plans of (t, l, .)
    (P:651-656); the kernel receives the (t, l, h) skip list at launch.

Every arithmetic step is a libcsa.so call (csa_calib_accumulate, csa_spatial_similarity,
csa_compile_plan, csa_build_work_list, csa_sparse_attn_fwd); this module only orders them, holds
the buffers and captures the per-step launch sequence in a CUDA graph (no host work between
layers at replay).  Cell convention (csa.h): cell = (t * L + l) * H + h.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Callable

import torch

from . import csa, ulysses
from .inputs import Layout

# "the same schedule for both 480p and 720p distilled LightX2V: A=0.763, C=0.863, k=5.64"
DISTILLED = (0.763, 0.863, 5.64)


def high_step_constants(n: int) -> tuple[float, float, float]:
    """(A(N), C, k) of the high-step regime, N = attention sequence length."""
    return 0.796 + 1.41e-6 * n, 0.99, 16.0


def epsilon_schedule(T: int, A: float, C: float, k: float) -> list[float]:
    """eps(t) = A + (C - A) exp(-k t / T), t = 0..T-1, t = 0 the highest noise (Eq.
    eq:epsilon_schedule).  Row a1: host fp64, passed to the kernel as a double."""
    return [A + (C - A) * math.exp(-k * t / T) for t in range(T)]


@dataclasses.dataclass
class PlanDictionary:
    """Compiled plans of all T * L * H cells (one csa.Plan) and the statistics behind them."""

    lay: Layout
    T: int
    L: int
    H: int
    plan: csa.Plan
    eps: list
    min_count: int
    prompts: int
    similarity: torch.Tensor   # fp64 [T * L * H]
    keep_count: torch.Tensor   # uint16 [T * L * H, N_B, N_Bkv]
    gamma: float = 0.87
    anchor_k: int = 5

    def cell_base(self, t: int, l: int) -> int:
        return (t * self.L + l) * self.H

    def shard(self, world: int, rank: int, perm: list | None = None) -> "PlanDictionary":
        """This rank's part of the dictionary for head-sharded inference: the cells
        (t, l, h) of heads perm[rank H/P:(rank+1) H/P] (default: contiguous heads), compiled by
        csa_compile_plan from those cells' keep counts and similarity -- cell-local, so every
        cell's plan is the full dictionary's bit for bit.  (Calibration itself is head-sharded
        with no collective: a rank can equally calibrate only its heads.)"""
        H = self.H
        if H % world:
            raise ValueError(f"{H} heads not divisible by {world} ranks")
        hp = H // world
        perm = list(range(H)) if perm is None else list(perm)
        mine = torch.tensor(perm[rank * hp:(rank + 1) * hp], device=self.keep_count.device)
        kc = self.keep_count.view(self.T * self.L, H, self.lay.NB, -1)
        keep = kc.view(torch.int16)[:, mine].contiguous().view(torch.uint16)
        sim = self.similarity.view(self.T * self.L, H)[:, mine].contiguous().view(-1)
        plan = csa.compile_plan(self.lay, keep.view(-1), self.min_count, similarity=sim,
                                gamma=self.gamma, anchor_k=self.anchor_k,
                                csr=self.plan.blk_idx.numel() > 0)
        return PlanDictionary(self.lay, self.T, self.L, hp, plan, self.eps, self.min_count,
                              self.prompts, sim, keep.view(-1, self.lay.NB, keep.shape[-1]),
                              self.gamma, self.anchor_k)

    def kept_fraction(self, t: int | None = None) -> float:
        """Kept area / dense area over the cells of timestep t (all cells if None)."""
        area = self.plan.kept_area.view(self.T, self.L * self.H)
        sel = area if t is None else area[t:t + 1]
        return float(sel.sum().item()) / (sel.numel() * float(self.lay.N) ** 2)


def calibrate(lay: Layout, T: int, L: int, H: int, prompts: int,
              qk_fn: Callable[[int, int, int], tuple[torch.Tensor, torch.Tensor]],
              constants: tuple[float, float, float], rho: float = 0.5, gamma: float = 0.87,
              anchor_k: int = 5, device="cuda", csr: bool = True,
              heads: list | None = None) -> PlanDictionary:
    """Offline calibration of the whole dictionary.

    qk_fn(prompt, t, l) -> conditional-branch Q, K bf16 [1, N, H, d] of that layer at that step.
    Per (prompt, t, l): one csa_calib_accumulate_sim pass adds the prompt's per-row selections at
    eps(t) to the cells' keep counts (a2-a5) and its cosines to the similarity sums (f1).  Then s = sim_sum / (F H |D|), min_count = ceil(rho |D|) and one csa_compile_plan over
    every cell (a6; s > gamma -> REPETITIVE).  csr=False: an intervals-only dictionary (the
    kernels walk the 1-D skip lists; 0.24 of the CSR plan bytes at Wan 720p: the
    mask bits and row pointers remain).

    heads: head-sharded calibration (BASELINE configs[4]) -- this rank calibrates and
    compiles only the cells of these heads of qk_fn's H (in this order), with no collective; the
    result equals calibrate(...).shard(P, r, perm) bit for bit (every step is cell-local)."""
    eps = epsilon_schedule(T, *constants)
    nb, nbk = lay.NB, lay.NBK  # query blocks x key blocks (non-square B_q x B_kv: P:1294-1328)
    sel = None
    if heads is not None:
        sel = torch.tensor(list(heads), dtype=torch.long, device=device)
        H = len(heads)
    cells = T * L * H
    keep = torch.zeros(cells * nb * nbk, dtype=torch.int16, device=device).view(torch.uint16)
    sim_sum = torch.zeros(cells, dtype=torch.float64, device=device)
    per = H * nb * nbk
    for p in range(prompts):
        for t in range(T):
            for l in range(L):
                q, k = qk_fn(p, t, l)
                if sel is not None:  # this rank's heads (a model's head-sharded projections)
                    q, k = q.index_select(2, sel), k.index_select(2, sel)
                c0 = (t * L + l) * H
                csa.calib_accumulate_sim(lay, q, k, eps[t],
                                         keep[c0 * nb * nbk:c0 * nb * nbk + per], anchor_k,
                                         sim_sum[c0:c0 + H])
    # smallest integer >= rho |D| (Eq. eq:mask_threshold in count space, reading Q6)
    min_count = math.ceil(rho * prompts - 1e-12)
    s = sim_sum / float(lay.F * lay.H * prompts)
    plan = csa.compile_plan(lay, keep, min_count, similarity=s, gamma=gamma, anchor_k=anchor_k,
                            csr=csr)
    return PlanDictionary(lay, T, L, H, plan, eps, min_count, prompts, s,
                          keep.view(cells, nb, nbk), gamma, anchor_k)


class DenoiseStep:
    """Attention of all L layers of one denoising step: layer l reads q[l % S], k[l % S],
    v[l % S] and writes o[l % S] (S buffer sets, [batch, N, H, d] bf16; batch 2 = the CFG
    branches sharing every cell plan), with the cell plans of (t, l, .).

    Work lists are built once per (t, l).  run(t) launches the L attention calls eagerly;
    capture(t) records the same sequence in a CUDA graph and replay(t) launches it (one host call
    per step; the dynamic scheduler's counters self-reset, so replays are independent)."""

    def __init__(self, dic: PlanDictionary, q: list, k: list, v: list, o: list):
        self.dic, self.q, self.k, self.v, self.o = dic, q, k, v, o
        self.work = [[csa.build_work_list(dic.plan, dic.cell_base(t, l), dic.H)
                      for l in range(dic.L)] for t in range(dic.T)]
        self.graphs: dict = {}
        self.stream = torch.cuda.Stream(device=q[0].device)

    def _launch(self, t: int, stream) -> None:
        dic, S = self.dic, len(self.q)
        for l in range(dic.L):
            s = l % S
            csa.sparse_attn_fwd(self.q[s], self.k[s], self.v[s], dic.plan, self.work[t][l],
                                cell_base=dic.cell_base(t, l), out=self.o[s], stream=stream)

    def run(self, t: int) -> None:
        self._launch(t, torch.cuda.current_stream())

    def capture(self, t: int) -> torch.cuda.CUDAGraph:
        if t not in self.graphs:
            with torch.cuda.stream(self.stream):
                self._launch(t, self.stream)  # warm: workspaces allocated, kernels loaded
            self.stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                self._launch(t, self.stream)
            self.graphs[t] = g
        return self.graphs[t]

    def replay(self, t: int) -> None:
        self.capture(t).replay()

    def flop(self, t: int) -> float:
        """Algorithmic FLOPs of step t: 4 d batch sum over its cells of kept_area."""
        d, b = self.q[0].shape[3], self.q[0].shape[0]
        area = self.dic.plan.kept_area.view(self.dic.T, -1)[t]
        return 4.0 * d * b * float(area.sum().item())


class ShardedDenoiseStep:
    """One denoising step of L attention layers head-sharded over the P ranks of a process group
    (SURVEY 8.6 / f4 on N GPUs).  Activations are sequence-sharded: layer l reads q[l % S],
    k[l % S], v[l % S] ([B, N/P, H, d], heads in the exchange order the rank dictionary was
    sharded with) and writes o[l % S].  Per layer: ONE stacked Q/K/V all-to-all per head chunk
    (ulysses.LayerExchange: the kernel reads the receive buffer and writes the return send
    buffer in place), csa_sparse_attn_fwd over the rank's cells (t, l, chunk heads) with both
    CFG branches in one launch (batch 2), the return all-to-all; with chunks > 1 the
    exchange of chunk c+1 overlaps the attention of chunk c (communication stream).  A DiT's
    layer l+1 reads layer l's output, so the overlap that exists is inside a layer (between head
    chunks) -- layers run in order.  run(t) launches eagerly; capture(t) records the whole step,
    NCCL calls included, in one CUDA graph.

    attention(t, l, c, q, k, v, out) replaces the kernel call (CPU gloo rehearsal of the schedule
    in tests/: the oracle stands in for the kernel); default: csa_sparse_attn_fwd.

    fused_out=True (CUDA, one head chunk): the return all-to-all is fused into the attention
    epilogue (ulysses.make_layer_step_fused_out, csa_sparse_attn_fwd_scatter): the layer outputs
    are symmetric-memory buffers owned by the step -- self.o[s] replaces the caller's o[s] (pass
    o=None) -- written by every rank's kernel directly."""

    def __init__(self, dic_rank: PlanDictionary | None, world: int, q: list, k: list, v: list,
                 o: list | None, chunks: int = 1, group=None, attention=None,
                 T: int | None = None, L: int | None = None, fused_out: bool = False):
        self.dic, self.world, self.chunks, self.group = dic_rank, world, chunks, group
        self.T = dic_rank.T if dic_rank is not None else T
        self.L = dic_rank.L if dic_rank is not None else L
        h = q[0].shape[2]
        self.hp = h // world
        if self.hp % chunks:
            raise ValueError(f"{self.hp} heads per rank not divisible into {chunks} chunks")
        self.hc = self.hp // chunks
        self.cur = (0, 0)
        cuda = q[0].is_cuda
        library_kernel = attention is None
        if attention is None:
            if dic_rank is None or dic_rank.H != self.hp:
                raise ValueError("the rank dictionary must hold H/P heads per (t, l)")
            self.work = [[[csa.build_work_list(dic_rank.plan, dic_rank.cell_base(t, l) + c * self.hc,
                                               self.hc)
                           for c in range(chunks)] for l in range(self.L)] for t in range(self.T)]
            attention = self._kernel
        self.attention = attention
        self.stream = torch.cuda.Stream(device=q[0].device) if cuda else None
        comm = torch.cuda.Stream(device=q[0].device) if cuda else None

        def attn(c, qh, kh, vh, out):
            t, l = self.cur
            self.attention(t, l, c, qh, kh, vh, out)

        if fused_out:
            if not cuda or chunks != 1 or not library_kernel:
                raise ValueError("fused_out: CUDA tensors, chunks = 1, the library kernel")

            def attn_scatter(qh, kh, vh, ptrs, recv):
                t, l = self.cur
                csa.sparse_attn_fwd_scatter(qh, kh, vh, self.dic.plan, self.work[t][l][0], ptrs,
                                            recv, cell_base=self.dic.cell_base(t, l))

            self.steps, self.o = [], []
            for s_ in range(len(q)):
                st = ulysses.make_layer_step_fused_out(q[s_], k[s_], v[s_], world, attn_scatter,
                                                       group=group)
                self.steps.append(st)
                self.o.append(st.out)
        else:
            self.steps = [ulysses.make_layer_step_chunked(q[s_], k[s_], v[s_], world, attn,
                                                          chunks, group=group, out=o[s_],
                                                          comm=comm)
                          for s_ in range(len(q))]
            self.o = o
        self.graphs: dict = {}

    def _kernel(self, t, l, c, qh, kh, vh, out):
        dic = self.dic
        csa.sparse_attn_fwd(qh, kh, vh, dic.plan, self.work[t][l][c],
                            cell_base=dic.cell_base(t, l) + c * self.hc, out=out)

    def _launch(self, t: int) -> None:
        S = len(self.steps)
        for l in range(self.L):
            self.cur = (t, l)
            self.steps[l % S]()

    def run(self, t: int) -> None:
        self._launch(t)

    def capture(self, t: int) -> torch.cuda.CUDAGraph:
        if t not in self.graphs:
            with torch.cuda.stream(self.stream):
                self._launch(t)  # warm: workspaces allocated, NCCL communicators up
            self.stream.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=self.stream):
                self._launch(t)
            self.graphs[t] = g
        return self.graphs[t]

    def replay(self, t: int) -> None:
        self.capture(t).replay()
