"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle's tests.

This module holds NO arithmetic of the method (no softmax, no energy, no selection, no plan
compilation).  It only produces:

* video-token geometry (``Layout``: F x H x W tokens, block size B);
* bf16 Q/K/V tensors with the shapes of the paper's workloads (``qkv``, ``structured_qk``);
* synthetic keep-count tensors (``synthetic_counts``) standing in for calibrated statistics at a
  target block sparsity -- they are *inputs* to ``csa_compile_plan`` / the oracle compiler;
* the hand-written tiny mask of BASELINE.json configs[0].

Recipes are stated in DESIGN.md section "Input recipe".  Every generator is a pure function of
its seed (torch Philox on the target device, or numpy PCG64 on the host).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch


@dataclasses.dataclass(frozen=True)
class Layout:
    """Spatiotemporal token grid partitioned in B-token blocks; BK > 0
    selects non-square B_q x B_kv = B x BK blocks: plan rows are the NB query
    blocks, plan columns the NBK key blocks."""

    F: int
    H: int
    W: int
    B: int = 128
    BK: int = 0

    @property
    def N(self) -> int:
        return self.F * self.H * self.W

    @property
    def NB(self) -> int:
        return (self.N + self.B - 1) // self.B

    @property
    def Bkv(self) -> int:
        return self.BK if self.BK > 0 else self.B

    @property
    def NBK(self) -> int:
        return (self.N + self.Bkv - 1) // self.Bkv

    def block_size(self, r: int) -> int:
        return min((r + 1) * self.B, self.N) - r * self.B

    def key_block_size(self, c: int) -> int:
        return min((c + 1) * self.Bkv, self.N) - c * self.Bkv


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    layout: Layout
    heads: int
    d: int
    sparsity: float | None  # target area sparsity of the synthetic plan (None: hand / calibrated)
    batch: int = 1


# BASELINE.json configs.  Geometry: P:1137-1139 (21x30x52 = 32760), P:916 (N = 75600 at 720p);
# heads / d: P:1152 (40 heads, d = 128); block 128: P:735.  Mochi geometry 28x30x53 (BASELINE
# "~44.5k"), 24 heads (EXT).
CONFIGS = {
    "tiny": Config("tiny", Layout(4, 8, 8, 64), 1, 64, None),
    "tiny_ragged": Config("tiny_ragged", Layout(2, 5, 25, 64), 1, 64, None),
    "wan480": Config("wan480", Layout(21, 30, 52, 128), 40, 128, 0.68),
    "wan720": Config("wan720", Layout(21, 45, 80, 128), 40, 128, 0.625),
    "mochi": Config("mochi", Layout(28, 30, 53, 128), 24, 128, None),
    "mochi85": Config("mochi85", Layout(15, 30, 53, 128), 24, 128, None),
}

# SURVEY 8.5 M1 hand mask (rows r0..r3 of N_B = 4): multi-interval rows, first/last columns.
TINY_HAND_MASK = np.array(
    [[1, 0, 0, 1],
     [1, 1, 0, 0],
     [0, 1, 1, 0],
     [1, 0, 1, 1]], dtype=np.uint8)


def qkv(batch: int, n: int, heads: int, d: int, seed: int, device="cpu",
        dtype=torch.bfloat16, std: float = 1.0):
    """Q, K, V ~ N(0, std^2) cast to bf16, layout [batch, N, heads, d] ("bshd").

    Seeds seed, seed+1, seed+2 (torch Philox on ``device``)."""
    out = []
    for s in range(3):
        g = torch.Generator(device=device)
        g.manual_seed(int(seed) * 1000003 + s)
        t = torch.randn((batch, n, heads, d), generator=g, device=device, dtype=torch.float32)
        if std != 1.0:
            t.mul_(std)
        out.append(t.to(dtype))
    return out


def structured_qk(lay: Layout, heads: int, d: int, head_seed: int, prompt_seed: int,
                  alpha, repetitive=(), device="cpu", tau_f: float = 2.0, tau_s: float = 3.0,
                  noise: float = 0.1):
    """Generator G: random-Fourier-feature Q/K realising a Gaussian spatiotemporal
    locality kernel (Obs. 1, 3, 4), a sink direction, prompt noise.

    alpha: scalar or per-head sequence (peak logit scale).  ``repetitive``: heads whose queries
    ignore the spatial-row coordinate (Obs. 4).  Returns Q, K, V bf16 [1, N, heads, d]."""
    n = lay.N
    nf = (d - 16) // 2
    alphas = np.broadcast_to(np.asarray(alpha, dtype=np.float64), (heads,))
    f = torch.arange(lay.F, device=device, dtype=torch.float32).repeat_interleave(lay.H * lay.W)
    i = torch.arange(lay.H, device=device, dtype=torch.float32).repeat_interleave(lay.W).repeat(lay.F)
    j = torch.arange(lay.W, device=device, dtype=torch.float32).repeat(lay.F * lay.H)
    pk = torch.stack([f / tau_f, i / tau_s, j / tau_s], dim=1)  # [N, 3]
    q = torch.zeros((n, heads, d), device=device, dtype=torch.float32)
    k = torch.zeros((n, heads, d), device=device, dtype=torch.float32)
    for h in range(heads):
        g = torch.Generator(device=device)
        g.manual_seed(int(head_seed) * 7919 + h)
        omega = torch.randn((nf, 3), generator=g, device=device)
        pq = pk.clone()
        if h in repetitive:
            pq[:, 1] = 0.0
        a = float(alphas[h])
        ph_q = pq @ omega.T
        ph_k = pk @ omega.T
        q[:, h, 0:2 * nf:2] = a * torch.cos(ph_q)
        q[:, h, 1:2 * nf:2] = a * torch.sin(ph_q)
        k[:, h, 0:2 * nf:2] = a * torch.cos(ph_k)
        k[:, h, 1:2 * nf:2] = a * torch.sin(ph_k)
        # sink direction in column 2*nf: every query leans on it, 4 seeded keys carry it
        q[:, h, 2 * nf] = 0.5
        sinks = torch.randint(0, n, (4,), generator=g, device=device)
        k[sinks, h, 2 * nf] = 3.0 * math.sqrt(d)
    g = torch.Generator(device=device)
    g.manual_seed(int(prompt_seed) * 104729 + 17)
    q += noise * torch.randn(q.shape, generator=g, device=device)
    k += noise * torch.randn(k.shape, generator=g, device=device)
    v = torch.randn(q.shape, generator=g, device=device)
    return (q.unsqueeze(0).to(torch.bfloat16), k.unsqueeze(0).to(torch.bfloat16),
            v.unsqueeze(0).to(torch.bfloat16))


def _block_centres(lay: Layout, block: int | None = None) -> np.ndarray:
    b = lay.B if block is None else block
    nb = (lay.N + b - 1) // b
    c = np.arange(nb)
    size = np.minimum((c + 1) * b, lay.N) - c * b
    tok = c * b + (size - 1) // 2
    f = tok // (lay.H * lay.W)
    i = (tok // lay.W) % lay.H
    j = tok % lay.W
    return np.stack([f, i, j], axis=1).astype(np.float64)


def synthetic_masks(lay: Layout, heads: int, target_sparsity: float, seed: int = 0,
                    lam_t: float = 1.0, tol: float = 0.005) -> np.ndarray:
    """Generator S: per-head block masks at a target area sparsity.

    Block (r, c) distance D = lam_t |f_r - f_c| + ||(i,j)_r - (i,j)_c|| / H between block-centre
    tokens; head keep fraction kappa_h ~ Beta(2,3); row fraction kappa_{h,r} = clip(m kappa_h
    exp(0.3 z), 1/N_Bkv, 1); keep the ceil(kappa N_Bkv) nearest key blocks (ties c asc) plus the
    key block holding the query block's centre token (the diagonal) and key block 0 (sink);
    bisect the global multiplier m until area sparsity is within tol of the target.
    Non-square layouts (lay.BK): rows are query blocks of B, columns key blocks of
    B_kv.  Returns uint8 [heads, N_B, N_Bkv]."""
    nb, nbk, rng = lay.NB, lay.NBK, np.random.default_rng(seed)
    cen = _block_centres(lay)
    ckey = _block_centres(lay, lay.Bkv)
    df = np.abs(cen[:, None, 0] - ckey[None, :, 0])
    ds = np.hypot(cen[:, None, 1] - ckey[None, :, 1], cen[:, None, 2] - ckey[None, :, 2]) / lay.H
    dist = lam_t * df + ds
    order = np.argsort(dist, axis=1, kind="stable")                   # [nb, nbk]
    qsizes = np.array([lay.block_size(r) for r in range(nb)], np.int64)
    ksizes = np.array([lay.key_block_size(c) for c in range(nbk)], np.int64)
    csum = np.concatenate([np.zeros((nb, 1), np.int64), np.cumsum(ksizes[order], axis=1)], axis=1)
    rows = np.arange(nb)
    rank = np.empty_like(order)
    rank[rows[:, None], order] = np.arange(nbk)[None, :]
    diag_c = (rows * lay.B + (qsizes - 1) // 2) // lay.Bkv             # = r for square blocks
    rank_diag = rank[rows, diag_c]
    rank_zero = rank[:, 0]
    kap_h = rng.beta(2.0, 3.0, size=heads)
    z = rng.standard_normal((heads, nb))

    def counts_for(m):
        kap = np.clip(m * kap_h[:, None] * np.exp(0.3 * z), 1.0 / nbk, 1.0)
        return np.minimum(np.ceil(kap * nbk).astype(np.int64), nbk)

    def sparsity_for(m):
        kk = counts_for(m)
        area_cols = csum[rows[None, :], kk]                            # [heads, nb]
        extra_d = np.where(rank_diag[None, :] >= kk, ksizes[diag_c][None, :], 0)
        extra_0 = np.where((rank_zero[None, :] >= kk) & (diag_c[None, :] != 0), ksizes[0], 0)
        area = ((area_cols + extra_d + extra_0) * qsizes[None, :]).sum()
        return 1.0 - area / float(heads * lay.N * lay.N)

    lo, hi = 1e-4, 50.0
    m = 1.0
    for _ in range(200):
        m = 0.5 * (lo + hi)
        s = sparsity_for(m)
        if abs(s - target_sparsity) <= tol * 0.2:
            break
        if s > target_sparsity:
            lo = m
        else:
            hi = m
    kk = counts_for(m)
    masks = np.zeros((heads, nb, nbk), np.uint8)
    for h in range(heads):
        sel = np.arange(nbk)[None, :] < kk[h][:, None]                # [nb, nbk] in rank space
        mh = np.zeros((nb, nbk), np.uint8)
        mh[rows[:, None], order] = sel
        mh[rows, diag_c] = 1
        mh[:, 0] = 1
        masks[h] = mh
    return masks


def synthetic_counts(lay: Layout, heads: int, target_sparsity: float, n_prompts: int = 64,
                     seed: int = 0) -> np.ndarray:
    """Keep counts consistent with a fully agreeing calibration set: |D| * M (uint16)."""
    return synthetic_masks(lay, heads, target_sparsity, seed).astype(np.uint16) * np.uint16(n_prompts)


def random_counts(nb: int, cells: int, n_prompts: int, seed: int, p_zero: float = 0.3,
                  nbk: int | None = None) -> np.ndarray:
    """Uniform random keep counts in [0, |D|] with extra zeros (plan-compiler edge coverage);
    [cells, nb, nbk] (nbk: key blocks of a non-square layout, default nb)."""
    rng = np.random.default_rng(seed)
    c = rng.integers(0, n_prompts + 1, size=(cells, nb, nb if nbk is None else nbk))
    c[rng.random(c.shape) < p_zero] = 0
    return c.astype(np.uint16)
