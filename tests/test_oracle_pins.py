"""Pins for the fp64 oracle (CPU only).  Each test fixes an oracle function against something
other than itself: NumPy/SciPy brute force with a materialised P, a library routine (torch SDPA
in fp64), a closed form, an invariant, or a value the paper prints (tests/golden/*, cited).
Each pin is chosen so a plausible slip (dropped term, wrong sign/index, transposed operand,
off-by-one block edge) fails it."""
import itertools
import math

import numpy as np
import pytest
import scipy.special
import torch

from conftest import golden_lines
from paper_2603_05503_b200 import inputs


def _rand(n, d, seed):
    rng = np.random.default_rng(seed)
    return rng.standard_normal((n, d)), rng.standard_normal((n, d)), rng.standard_normal((n, d))


def _block_of(n, b):
    return np.arange(n) // b


def brute_masked(q, k, v, scale, b, mask):
    """Materialised P with -inf outside kept blocks, SciPy softmax (independent of the oracle)."""
    n = q.shape[0]
    logits = scale * (q @ k.T)
    if mask is not None:
        blk = _block_of(n, b)
        keep = mask[blk[:, None], blk[None, :]].astype(bool)
        logits = np.where(keep, logits, -np.inf)
    p = scipy.special.softmax(logits, axis=1)
    return p @ v, scipy.special.logsumexp(logits, axis=1), p


# ---------------------------------------------------------------- a7: masked attention
@pytest.mark.parametrize("n,b,d", [(256, 64, 64), (250, 64, 64), (200, 32, 16)])
def test_masked_attention_equals_brute_force(orc, n, b, d):
    q, k, v = _rand(n, d, 1)
    nb = orc.num_blocks(n, b)
    rng = np.random.default_rng(7)
    mask = (rng.random((nb, nb)) < 0.5).astype(np.uint8)
    mask[np.arange(nb), np.arange(nb)] = 1
    if n == 256:
        mask = inputs.TINY_HAND_MASK.copy()
    scale = 1.0 / math.sqrt(d)
    out, lse = orc.masked_attention_rows(q, k, v, scale, b, mask)
    ref, ref_lse, p = brute_masked(q, k, v, scale, b, mask)
    assert np.max(np.abs(out - ref)) < 1e-12
    assert np.max(np.abs(lse - ref_lse)) < 1e-12
    # row sums over kept keys are 1 (P:505-507 'row ... sums up to 1' applied to kept support)
    logits = scale * (q @ k.T)
    blk = _block_of(n, b)
    keep = mask[blk[:, None], blk[None, :]].astype(bool)
    rs = np.where(keep, np.exp(logits - lse[:, None]), 0.0).sum(axis=1)
    assert np.max(np.abs(rs - 1.0)) < 1e-12
    # each output coordinate lies in [min, max] of the kept V rows (convex combination)
    for i in range(0, n, 17):
        vk = v[keep[i]]
        assert np.all(out[i] <= vk.max(axis=0) + 1e-12) and np.all(out[i] >= vk.min(axis=0) - 1e-12)


def test_all_ones_mask_equals_library_dense_attention(orc):
    """All-ones plan == dense attention computed by torch SDPA in fp64."""
    n, d, b = 250, 64, 64
    q, k, v = _rand(n, d, 3)
    scale = 1.0 / math.sqrt(d)
    out, _ = orc.masked_attention_rows(q, k, v, scale, b, np.ones((4, 4), np.uint8))
    out2, _ = orc.masked_attention_rows(q, k, v, scale, b, None)
    t = lambda a: torch.from_numpy(a)[None, None]
    ref = torch.nn.functional.scaled_dot_product_attention(t(q), t(k), t(v), scale=scale)[0, 0].numpy()
    assert np.max(np.abs(out - ref)) < 1e-12
    assert np.array_equal(out, out2)


def test_exact_block_structure_sparse_equals_dense(orc):
    """Logits ~ -inf outside a block pattern + the matching mask -> sparse == dense."""
    n, b, d = 256, 64, 64
    nb = 4
    mask = inputs.TINY_HAND_MASK
    rng = np.random.default_rng(5)
    A = math.sqrt(90.0 * math.sqrt(d))  # sigma*A^2 = 90: off-pattern weight e^-90 relative
    blk = _block_of(n, b)
    q = 0.05 * rng.standard_normal((n, d))
    k = 0.05 * rng.standard_normal((n, d))
    q[:, :nb] += A * mask[blk]                    # row r's indicator of kept columns
    k[:, :nb] += A * np.eye(nb)[blk]               # column c's one-hot
    v = rng.standard_normal((n, d))
    scale = 1.0 / math.sqrt(d)
    sparse, _ = orc.masked_attention_rows(q, k, v, scale, b, mask)
    dense, _ = orc.masked_attention_rows(q, k, v, scale, b, None)
    assert np.max(np.abs(sparse - dense)) < 1e-12


def test_single_block_row_is_convex_combination_of_that_block(orc):
    n, b, d = 256, 64, 8
    q, k, v = _rand(n, d, 9)
    mask = np.eye(4, dtype=np.uint8)[[2, 0, 3, 1]]
    out, _ = orc.masked_attention_rows(q, k, v, 0.3, b, mask)
    for i in range(n):
        c = int(np.argmax(mask[i // b]))
        vb = v[c * b:(c + 1) * b]
        assert np.all(out[i] <= vb.max(0) + 1e-12) and np.all(out[i] >= vb.min(0) - 1e-12)


# ---------------------------------------------------------------- a8: anchor rows
def test_anchor_rows_and_nearest(orc):
    for line in golden_lines("worked_examples.txt"):
        if line.startswith("anchors"):
            lhs, rhs = line.split("|")
            _, H, kA = lhs.split()
            assert orc.anchor_rows(int(H), int(kA)) == [int(x) for x in rhs.split()]
    assert orc.anchor_rows(30, 30) == list(range(30))
    # brute-force nearest with explicit tie rule (lower anchor)
    for H in (1, 5, 8, 30, 45):
        for kA in range(1, H + 1):
            a = orc.anchor_rows(H, kA)
            for i in range(H):
                dist = [abs(i - x) for x in a]
                assert orc.nearest_anchor(H, kA, i) == dist.index(min(dist))
            # max distance bound of a centred equispaced placement
            assert max(min(abs(i - x) for x in a) for i in range(H)) <= math.ceil(H / (2 * kA))


def test_anchor_sparsity_matches_paper_table(orc):
    """1 - k/H reproduces Table tab:anchor_bench's sparsity column."""
    H = 30
    n = 21 * 30 * 52
    for line in golden_lines("anchor_bench_sparsity.txt"):
        kA, pct = line.split()
        kA = int(kA)
        # kept area of a REPETITIVE cell: F*k*W queries x N keys
        cell = orc.compile_cell(np.zeros((256, 256)), n, 128, 21, H, 52, 1, similarity=1.0,
                                gamma=0.87, anchor_k=kA)
        assert cell["kind"] == 1
        assert round(100 * orc.sparsity_of_cell(cell["kept_area"], n), 1) == float(pct)


def test_anchor_k_equals_H_is_dense_and_repetitive_workload_exact(orc):
    F, H, W, d = 2, 6, 5, 8
    n = F * H * W
    q, k, v = _rand(n, d, 11)
    dense, _ = orc.masked_attention_rows(q, k, v, 0.4, 64, None)
    full, _ = orc.anchor_attention_rows(F, H, W, q, k, v, 0.4, H)
    assert np.max(np.abs(full - dense)) < 1e-14
    # queries depending only on (f, j): every spatial row is identical -> anchors exact
    rng = np.random.default_rng(3)
    base = rng.standard_normal((F, 1, W, d))
    qr = np.broadcast_to(base, (F, H, W, d)).reshape(n, d)
    dense_r, _ = orc.masked_attention_rows(qr, k, v, 0.4, 64, None)
    for kA in (1, 2, 5):
        out, _ = orc.anchor_attention_rows(F, H, W, qr, k, v, 0.4, kA)
        assert np.max(np.abs(out - dense_r)) < 1e-12


def test_anchor_broadcast_is_positionwise_copy_of_nearest_anchor(orc):
    F, H, W, d = 2, 7, 4, 4
    n = F * H * W
    q, k, v = _rand(n, d, 12)
    out, _ = orc.anchor_attention_rows(F, H, W, q, k, v, 0.5, 3)
    dense, _ = orc.masked_attention_rows(q, k, v, 0.5, 64, None)
    a = orc.anchor_rows(H, 3)
    for f in range(F):
        for i in range(H):
            m = orc.nearest_anchor(H, 3, i)
            for j in range(W):
                t = f * H * W + i * W + j
                s = f * H * W + a[m] * W + j
                assert np.array_equal(out[t], out[s])
                assert np.max(np.abs(out[t] - dense[s])) < 1e-14


# ---------------------------------------------------------------- a2/a3: LSE and block energy
def test_lse_and_energy_against_materialised_P(orc):
    n, b, d = 250, 64, 16
    q, k, _ = _rand(n, d, 21)
    scale = 0.7
    lse = orc.row_lse(q, k, scale)
    assert np.max(np.abs(lse - scipy.special.logsumexp(scale * q @ k.T, axis=1))) < 1e-12
    E = orc.block_energy(q, k, scale, b)
    p = scipy.special.softmax(scale * q @ k.T, axis=1)
    nb = 4
    ref = np.zeros((nb, nb))
    for r in range(nb):
        rows = slice(r * b, min((r + 1) * b, n))
        for c in range(nb):
            ref[r, c] = p[rows, c * b:min((c + 1) * b, n)].sum() / p[rows].shape[0]
    assert np.max(np.abs(E - ref)) < 1e-12
    assert np.max(np.abs(E.sum(axis=1) - 1.0)) < 1e-12      # P:507 rows sum to 1 (ragged too)
    E2 = orc.block_energy(q, k, scale, b, lse=lse)
    assert np.max(np.abs(E2 - E)) < 1e-15


def test_energy_uniform_and_block_diagonal_closed_forms(orc):
    n, b, d = 250, 64, 16
    # q = 0 -> every P_ij = 1/N -> E_rc = |J_c| / N
    q = np.zeros((n, d))
    k = np.random.default_rng(1).standard_normal((n, d))
    E = orc.block_energy(q, k, 1.0, b)
    sizes = np.array([64, 64, 64, 58])
    assert np.max(np.abs(E - sizes[None, :] / n)) < 1e-15
    # block-diagonal P (each query attends inside its own block) -> E = I
    blk = _block_of(n, b)
    A = math.sqrt(200.0)
    q = np.zeros((n, d)); k = np.zeros((n, d))
    q[:, :4] = A * np.eye(4)[blk]
    k[:, :4] = A * np.eye(4)[blk]
    E = orc.block_energy(q, k, 1.0, b)
    assert np.max(np.abs(E - np.eye(4))) < 1e-12


# ---------------------------------------------------------------- a4: selection
def test_selection_worked_examples(orc):
    for line in golden_lines("worked_examples.txt"):
        if not line.startswith("select"):
            continue
        lhs, e, kept = line.split("|")
        eps = float(lhs.split()[1])
        e = np.array([float(x) for x in e.split()])
        exp = np.zeros(e.size, np.uint8)
        exp[[int(x) for x in kept.split()]] = 1
        assert np.array_equal(orc.select(e, eps), exp)


def test_selection_is_minimal_against_subset_brute_force(orc):
    """Eq. eq:row_energy_constraint solved exactly (P:533 'optimally solves'), N_B <= 12."""
    rng = np.random.default_rng(0)
    for trial in range(300):
        nb = int(rng.integers(1, 11))
        e = rng.dirichlet(np.full(nb, rng.uniform(0.2, 3.0)))
        eps = float(rng.uniform(0.5, 0.999))
        kept = orc.select(e, eps)
        best = None
        for size in range(1, nb + 1):
            if any(e[list(s)].sum() >= eps for s in itertools.combinations(range(nb), size)):
                best = size
                break
        if best is None:          # unreachable eps (rounding) -> keep everything (Q5)
            assert kept.sum() == nb
        else:
            assert kept.sum() == best
            assert e[kept.astype(bool)].sum() >= eps
        assert kept.sum() >= 1


def test_selection_tie_order_and_prefix_monotone(orc):
    e = np.full(10, 0.1)
    assert list(np.nonzero(orc.select(e, 0.35))[0]) == [0, 1, 2, 3]
    rng = np.random.default_rng(4)
    e = rng.dirichlet(np.ones(30))
    prev = orc.select(e, 0.5)
    for eps in (0.6, 0.8, 0.9, 0.99):
        cur = orc.select(e, eps)
        assert np.all(cur >= prev)
        prev = cur


# ---------------------------------------------------------------- a1: eps schedule
def test_epsilon_schedule_paper_values(orc):
    for line in golden_lines("epsilon_schedule.txt"):
        name, n, T, A, C, k, t, val, tol = line.split()
        A = orc.A_of_N(float(n)) if A == "A(N)" else float(A)
        e = orc.epsilon(int(t), int(T), A, float(C), float(k))
        assert abs(e - float(val)) <= float(tol), name
    # closed form of the fitted level at the paper's geometry: 0.796 + 1.41e-6 * 32760
    assert abs(orc.A_of_N(32760) - 0.8421916) < 1e-12
    # non-increasing in t for C >= A, k >= 0
    A = orc.A_of_N(75600)
    seq = [orc.epsilon(t, 50, A, 0.99, 16) for t in range(50)]
    assert all(x >= y for x, y in zip(seq, seq[1:]))


# ---------------------------------------------------------------- a5/a6: counts and compile
def test_threshold_worked_examples_and_min_count(orc):
    assert orc.min_count(0.5, 64) == 32
    assert orc.min_count(0.6, 2) == 2 and orc.min_count(0.5, 2) == 1
    for line in golden_lines("worked_examples.txt"):
        if not line.startswith("threshold"):
            continue
        lhs, cnt, exp = line.split("|")
        _, nd, rho = lhs.split()
        cnt = np.array([int(x) for x in cnt.split()], np.uint16)
        nb = cnt.size
        counts = np.zeros((nb, nb), np.uint16)
        counts[:] = cnt
        cell = orc.compile_cell(counts, nb * 4, 4, 1, 1, nb * 4, orc.min_count(float(rho), int(nd)))
        assert list(cell["mask"][0]) == [int(x) for x in exp.split()]


def test_accumulate_is_count_of_kept(orc):
    rng = np.random.default_rng(1)
    masks = (rng.random((64, 5, 5)) < 0.4).astype(np.uint8)
    cnt = np.zeros((5, 5), np.uint16)
    for m in masks:
        orc.accumulate(m, cnt)
    assert np.array_equal(cnt, masks.sum(0))
    # mean >= rho <=> count >= min_count (Eq. eq:mask_mean / eq:mask_threshold)
    for rho in (0.1, 0.5, 0.77, 1.0):
        mc = orc.min_count(rho, 64)
        assert np.array_equal(cnt >= mc, masks.mean(0) >= rho)


def _decode(iv, nb):
    row = np.zeros(nb, np.uint8)
    for s, e in iv:
        row[s:e] = 1
    return row


def test_intervals_worked_examples_and_round_trip(orc):
    for line in golden_lines("worked_examples.txt"):
        if not line.startswith("intervals"):
            continue
        _, bits, exp = line.split("|")
        bits = np.array([int(x) for x in bits.split()], np.uint16)
        nb = bits.size
        counts = np.tile(bits, (nb, 1))
        cell = orc.compile_cell(counts, nb * 2, 2, 1, 1, nb * 2, 1)
        got = cell["ivl"][cell["ivl_row_ptr"][0]:cell["ivl_row_ptr"][1]].ravel().tolist()
        assert got == [int(x) for x in exp.split()]
    rng = np.random.default_rng(2)
    for trial in range(200):
        nb = int(rng.integers(1, 40))
        counts = (rng.random((nb, nb)) < rng.random()).astype(np.uint16) * 3
        cell = orc.compile_cell(counts, nb * 8 - int(rng.integers(0, 8)), 8, 1, 1, 1, 2)
        mask = cell["mask"]
        for r in range(nb):
            iv = cell["ivl"][cell["ivl_row_ptr"][r]:cell["ivl_row_ptr"][r + 1]]
            assert np.array_equal(_decode(iv, nb), mask[r])            # decode(compile) = id
            assert all(iv[x][1] < iv[x + 1][0] for x in range(len(iv) - 1))  # non-adjacent
            idx = cell["blk_idx"][cell["blk_row_ptr"][r]:cell["blk_row_ptr"][r + 1]]
            assert list(idx) == list(np.nonzero(mask[r])[0])
            if counts[r].max() < 2:                                     # repaired row (Q7)
                assert mask[r].sum() == 1 and mask[r][int(np.argmax(counts[r]))] == 1
            else:
                assert np.array_equal(mask[r], (counts[r] >= 2).astype(np.uint8))


def test_area_and_repetitive_rule(orc):
    n, b = 4 * 64, 64
    cell = orc.compile_cell(np.eye(4, dtype=np.uint16), n, b, 4, 8, 8, 1)
    assert orc.sparsity_of_cell(cell["kept_area"], n) == 0.75
    ragged = orc.compile_cell(np.ones((4, 4), np.uint16), 250, 64, 2, 5, 25, 1)
    assert ragged["kept_area"] == 250 * 250                              # all-ones = N^2
    z = np.ones((4, 4), np.uint16)
    assert orc.compile_cell(z, 256, 64, 4, 8, 8, 1, similarity=0.87, gamma=0.87)["kind"] == 0
    rep = orc.compile_cell(z, 256, 64, 4, 8, 8, 1, similarity=0.8700001, gamma=0.87, anchor_k=2)
    assert rep["kind"] == 1 and rep["kept_area"] == 4 * 2 * 8 * 256 and rep["blk_idx"].size == 0


def test_geometry(orc):
    for line in golden_lines("worked_examples.txt"):
        if line.startswith("token"):
            lhs, v = line.split("|")
            _, H, W, f, i, j = lhs.split()
            assert orc.token_index(int(H), int(W), int(f), int(i), int(j)) == int(v)
    assert orc.num_blocks(32760, 128) == 256 and 32760 - 255 * 128 == 120   # P:1139 ragged tail
    assert orc.num_blocks(75600, 128) == 591


_WL_KEYS = {  # the total orders csa.h states for csa_build_work_list, written out as sort keys
    0: lambda h, kind, idx, cost: (-cost, h, kind, idx),   # longest-first, ties (h, kind, idx)
    1: lambda h, kind, idx, cost: (h, kind, idx),          # natural
    2: lambda h, kind, idx, cost: (h, -cost, kind, idx),   # head-major, longest-first in a head
}


@pytest.mark.parametrize("order", [0, 1, 2])
@pytest.mark.parametrize("seed", [3, 4])
def test_work_list_is_sorted_permutation(orc, order, seed):
    """Every order is the enumeration of all items (MASK rows, REPETITIVE anchor tiles) sorted by
    its key, built here from scratch with Python's sorted(): a flipped comparison, a dropped
    tie-break or a missing item fails.  Costs drawn from a small range so ties are frequent."""
    rng = np.random.default_rng(seed)
    n, b, F, W = 250 * 4, 64, 2, 25
    nb = -(-n // b)
    kinds = np.array([0, 1, 0, 0, 1], np.uint8)
    ak = np.array([0, 2, 0, 0, 5], np.int32)
    nnz = rng.integers(1, 4, size=(kinds.size, nb)).astype(np.int32)
    wl = orc.work_list(n, b, F, W, kinds, ak, nnz, order=order)
    expect = []
    for h in range(kinds.size):
        if kinds[h]:
            for u in range(-(-F * int(ak[h]) * W // 128)):
                expect.append((h, 1, u, nb))
        else:
            for r in range(nb):
                expect.append((h, 0, r, int(nnz[h, r])))
    expect.sort(key=lambda t: _WL_KEYS[order](*t))
    got = [((int(c) >> 20) & 0x7FF, int(c) >> 31, int(c) & 0xFFFFF) for c in wl]
    assert got == [(h, kind, idx) for h, kind, idx, _ in expect]


def test_pair_work_list_covers_every_row_once(orc):
    """Order 3: item p of a head stands for members (2p, 2p+1); cost = members' sum."""
    rng = np.random.default_rng(8)
    n, b, F, W = 250 * 3, 64, 2, 25        # N_B = 12 (even) -- and an odd case below
    for n_, nb in ((n, 12), (250 * 3 - 64, 11)):
        kinds = np.array([0, 1, 0], np.uint8)
        ak = np.array([0, 3, 0], np.int32)
        nnz = rng.integers(1, nb + 1, size=(3, nb)).astype(np.int32)
        wl = orc.work_list(n_, b, F, W, kinds, ak, nnz, order=3)
        nu = (F * 3 * W + 127) // 128
        assert wl.size == 2 * ((nb + 1) // 2) + (nu + 1) // 2
        covered = []
        prev = None
        for code in wl:
            kind, h, p = int(code) >> 31, (int(code) >> 20) & 0x7FF, int(code) & 0xFFFFF
            units = nu if kind else nb
            members = [u for u in (2 * p, 2 * p + 1) if u < units]
            cost = nb * len(members) if kind else int(sum(nnz[h, u] for u in members))
            key = (h, -cost, p)
            assert prev is None or key > prev        # head-major, cost desc, p asc
            prev = key
            covered += [(h, u) for u in members]
        expect = [(h, u) for h in (0, 2) for u in range(nb)] + [(1, u) for u in range(nu)]
        assert sorted(covered) == sorted(expect)


# ---------------------------------------------------------------- f1: spatial similarity
def _brute_spatial_cos(F, H, W, q, k, scale, kA, anchors_near):
    """Materialised dense P (SciPy softmax), reshaped to [F, H, W, N]; Frobenius cosine of the
    W x N blocks of row i and of its nearest anchor row (independent of the oracle)."""
    p = scipy.special.softmax(scale * (q @ k.T), axis=1).reshape(F, H, W, -1)
    out = np.empty((F, H))
    for f in range(F):
        for i in range(H):
            a = anchors_near[i]
            x, y = p[f, i].ravel(), p[f, a].ravel()
            out[f, i] = x @ y / (np.linalg.norm(x) * np.linalg.norm(y))
    return out


def test_spatial_cos_equals_materialised_P(orc):
    F, H, W, d = 2, 7, 5, 16
    n = F * H * W
    q, k, _ = _rand(n, d, 31)
    for kA in (1, 3, 7):
        a = orc.anchor_rows(H, kA)
        near = [a[orc.nearest_anchor(H, kA, i)] for i in range(H)]
        ref = _brute_spatial_cos(F, H, W, q, k, 0.3, kA, near)
        got = np.array([[orc.spatial_cos(F, H, W, q, k, 0.3, kA, f, i) for i in range(H)]
                        for f in range(F)])
        assert np.max(np.abs(got - ref)) < 1e-12
        # anchor rows are their own nearest anchor: cos = 1
        for f in range(F):
            for m in a:
                assert abs(got[f, m] - 1.0) < 1e-14
        assert abs(orc.spatial_similarity(F, H, W, q, k, 0.3, kA) - ref.mean()) < 1e-12


def test_spatial_similarity_closed_forms(orc):
    F, H, W, d = 2, 6, 4, 48
    n = F * H * W
    # k = H: every row is an anchor -> s = 1
    q, k, _ = _rand(n, d, 32)
    assert abs(orc.spatial_similarity(F, H, W, q, k, 0.5, H) - 1.0) < 1e-14
    # queries independent of the spatial row (Obs. 4's ideal case) -> P^(f,i) = P^(f,a) -> s = 1
    rng = np.random.default_rng(4)
    base = rng.standard_normal((F, 1, W, d))
    qr = np.broadcast_to(base, (F, H, W, d)).reshape(n, d)
    for kA in (1, 2, 5):
        assert abs(orc.spatial_similarity(F, H, W, qr, k, 0.5, kA) - 1.0) < 1e-13
    # one-hot attention (query t attends to key t only): blocks of different rows are
    # orthogonal -> cos = 0 except on the k anchor rows -> s = k/H
    eye = 30.0 * np.eye(n, d)  # n = 48 <= d
    for kA in (1, 2, 3, 6):
        s = orc.spatial_similarity(F, H, W, eye, eye, 1.0, kA)
        assert abs(s - kA / H) < 1e-12


# ---------------------------------------------------------------- f2: plan compaction
def test_percentile_nearest_rank_textbook(orc):
    v = [15, 20, 35, 40, 50]  # the standard nearest-rank example
    assert [orc.percentile_nearest_rank(v, p) for p in (5, 30, 40, 50, 100)] == [15, 20, 20, 35, 50]
    assert orc.percentile_nearest_rank(list(range(1, 11)), 90) == 9
    assert orc.percentile_nearest_rank([7] * 3, 100) == 7


def test_merge_row_worked_example_and_ties(orc):
    assert orc.merge_row([(0, 2), (3, 4), (10, 12)], 2) == ([(0, 4), (10, 12)], 1)
    assert orc.merge_row([(0, 1), (2, 3), (4, 5)], 2) == ([(0, 3), (4, 5)], 1)      # tie: leftmost
    assert orc.merge_row([(0, 1), (5, 6)], 3) == ([(0, 1), (5, 6)], 0)              # within target
    assert orc.merge_row([(0, 1), (5, 6), (9, 10)], 1) == ([(0, 10)], 7)


def test_merge_row_is_optimal_against_subset_brute_force(orc):
    """Merging two adjacent intervals removes exactly the gap between them, so reaching `target`
    removes n - target gaps: the minimum total of added blocks is the sum of the n - target
    smallest gaps (checked by enumerating every gap subset), and the result must decode to a
    superset of the row with at most `target` intervals."""
    rng = np.random.default_rng(8)
    for _ in range(300):
        nb = int(rng.integers(4, 40))
        row = rng.random(nb) < rng.uniform(0.2, 0.7)
        row[int(rng.integers(nb))] = True
        ivl, c = [], 0
        while c < nb:
            if row[c]:
                s = c
                while c < nb and row[c]:
                    c += 1
                ivl.append((s, c))
            else:
                c += 1
        n = len(ivl)
        target = int(rng.integers(1, n + 1))
        merged, added = orc.merge_row(ivl, target)
        gaps = [ivl[i + 1][0] - ivl[i][1] for i in range(n - 1)]
        best = min((sum(gaps[i] for i in sub) for sub in itertools.combinations(range(n - 1), n - target)),
                   default=0)
        assert added == best and len(merged) == min(n, max(target, 1))
        kept = np.zeros(nb, bool)
        for s_, e_ in merged:
            kept[s_:e_] = True
        assert kept[row].all() and kept.sum() == row.sum() + added


def test_skipped_iou_and_timestep_clusters(orc):
    # skipped {(0,1),(0,2)} vs {(0,2),(1,3)} over a 2x4 mask -> 1/3
    k1 = np.ones((2, 4), np.uint8)
    k2 = np.ones((2, 4), np.uint8)
    k1[0, 1] = k1[0, 2] = 0
    k2[0, 2] = k2[1, 3] = 0
    assert orc.skipped_iou(k1, k2) == 1.0 / 3.0
    assert orc.skipped_iou(k1, k1) == 1.0
    assert orc.skipped_iou(np.ones(5), np.ones(5)) == 1.0  # nothing skipped
    a, b = np.array([0, 1, 1]), np.array([1, 0, 1])
    assert orc.skipped_iou(a, b) == 0.0
    # {t0, t1} mutually >= tau; t2 >= tau with t1 only; t3 isolated
    iou = np.eye(4)
    iou[0, 1] = iou[1, 0] = 0.99
    iou[1, 2] = iou[2, 1] = 0.99
    iou[0, 2] = iou[2, 0] = 0.5
    assert orc.cluster_timesteps(iou, 0.97).tolist() == [0, 0, 1, 2]
    assert orc.cluster_timesteps(np.ones((5, 5)), 0.98).tolist() == [0] * 5
    assert orc.cluster_timesteps(np.eye(4) * 0 + np.eye(4), 1.0).tolist() == [0, 1, 2, 3]


def test_timestep_clusters_are_cliques_and_greedy(orc):
    rng = np.random.default_rng(9)
    for _ in range(200):
        T = int(rng.integers(2, 12))
        m = rng.random((T, T))
        iou = (m + m.T) / 2
        np.fill_diagonal(iou, 1.0)
        tau = float(rng.uniform(0.3, 0.8))
        cl = orc.cluster_timesteps(iou, tau)
        for c in set(cl.tolist()):
            mem = np.flatnonzero(cl == c)
            assert all(iou[x, y] >= tau for x in mem for y in mem)
        # greedy: t could not join any cluster created before its own
        for t in range(T):
            for c in range(cl[t]):
                earlier = [u for u in range(t) if cl[u] == c]
                assert not all(iou[t, u] >= tau for u in earlier)


# ---------------------------------------------------------------- f3: non-square B_q x B_kv
def brute_masked_rect(q, k, v, scale, bq, bk, mask):
    """Token-level mask from a B_q x B_kv block mask, materialised softmax."""
    n = q.shape[0]
    keep = mask[_block_of(n, bq)[:, None], _block_of(n, bk)[None, :]].astype(bool)
    logits = np.where(keep, scale * (q @ k.T), -np.inf)
    return scipy.special.softmax(logits, axis=1) @ v, scipy.special.logsumexp(logits, axis=1), keep


@pytest.mark.parametrize("n,bq,bk", [(250, 64, 16), (250, 32, 48), (300, 128, 80), (130, 64, 192)])
def test_rect_masked_attention_equals_brute_force(orc, n, bq, bk):
    q, k, v = _rand(n, 16, 3)
    nbq, nbk = orc.num_blocks(n, bq), orc.num_blocks(n, bk)
    mask = (np.random.default_rng(5).random((nbq, nbk)) < 0.5).astype(np.uint8)
    mask[:, -1] = 1  # the ragged last key block kept somewhere; no empty row
    out, lse = orc.masked_attention_rows(q, k, v, 0.25, bq, mask, block_kv=bk)
    ref, ref_lse, keep = brute_masked_rect(q, k, v, 0.25, bq, bk, mask)
    assert np.max(np.abs(out - ref)) < 1e-12 and np.max(np.abs(lse - ref_lse)) < 1e-12
    rs = np.where(keep, np.exp(0.25 * (q @ k.T) - lse[:, None]), 0.0).sum(axis=1)
    assert np.max(np.abs(rs - 1.0)) < 1e-12


def test_rect_refinement_of_square_mask_is_identical(orc):
    """A 128 x 128 mask refined to 128 x 64 (every kept column c -> 2c, 2c+1) keeps the same key
    set: the rect oracle must give the square oracle's outputs bit for bit."""
    n, d = 600, 16
    q, k, v = _rand(n, d, 9)
    nb, nbk = orc.num_blocks(n, 128), orc.num_blocks(n, 64)
    sq = (np.random.default_rng(2).random((nb, nb)) < 0.5).astype(np.uint8)
    sq[np.arange(nb), np.arange(nb)] = 1
    rect = np.repeat(sq, 2, axis=1)[:, :nbk]
    a, la = orc.masked_attention_rows(q, k, v, 0.25, 128, sq)
    b, lb = orc.masked_attention_rows(q, k, v, 0.25, 128, rect, block_kv=64)
    assert np.array_equal(a, b) and np.array_equal(la, lb)
    dense, _ = orc.masked_attention_rows(q, k, v, 0.25, 128, None, block_kv=80)
    ones, _ = orc.masked_attention_rows(q, k, v, 0.25, 128, None)
    assert np.array_equal(dense, ones)  # no mask: every key, whatever the key block size


@pytest.mark.parametrize("n,bq,bk", [(75, 16, 8), (250, 128, 80), (333, 64, 112)])
def test_rect_compile_against_token_level_count(orc, n, bq, bk):
    """Threshold / repair / CSR / intervals / kept area of a B_q x B_kv cell against a direct
    token-level construction."""
    nbq, nbk = orc.num_blocks(n, bq), orc.num_blocks(n, bk)
    rng = np.random.default_rng(n)
    cnt = rng.integers(0, 9, size=(nbq, nbk)).astype(np.uint16)
    cnt[0] = 0  # emptied row -> repair keeps argmax (all zero: lowest c = 0)
    c = orc.compile_cell(cnt, n, bq, 1, 1, n, 5, block_kv=bk)
    m = (cnt >= 5).astype(np.uint8)
    m[0, 0] = 1
    assert np.array_equal(c["mask"], m)
    keep = m[_block_of(n, bq)[:, None], _block_of(n, bk)[None, :]]
    assert c["kept_area"] == int(keep.sum())
    rows = np.repeat(np.arange(nbq), m.sum(axis=1).astype(np.int64))
    assert np.array_equal(c["blk_idx"], np.nonzero(m)[1]) and len(rows) == c["blk_row_ptr"][-1]
    for r in range(nbq):
        ivl = c["ivl"][c["ivl_row_ptr"][r]:c["ivl_row_ptr"][r + 1]]
        dec = np.zeros(nbk, np.uint8)
        for s0, e0 in ivl:
            dec[s0:e0] = 1
        assert np.array_equal(dec, m[r])


def test_epsilon_schedules_paper_constants(orc):
    """P:886 distilled (A, C, k) = (0.763, 0.863, 5.64) and P:888-894 high-step constants through
    the oracle's Eq. eq:epsilon_schedule and the runtime's host schedule (row a1): eps(0) = C,
    strictly decreasing, above A, and eps(t) - A = (C - A) e^{-k t/T} (geometric ratio e^{-k/T})."""
    from paper_2603_05503_b200 import pipeline

    for consts, T in ((pipeline.DISTILLED, 4), (pipeline.high_step_constants(32760), 50)):
        A, C, k = consts
        host = pipeline.epsilon_schedule(T, A, C, k)
        ref = [orc.epsilon(t, T, A, C, k) for t in range(T)]
        assert np.allclose(host, ref, rtol=0, atol=1e-15)
        assert host[0] == C and all(a > b > A for a, b in zip(host, host[1:]))
        ratios = [(host[t + 1] - A) / (host[t] - A) for t in range(T - 1)]
        assert np.allclose(ratios, math.exp(-k / T), rtol=1e-12)
    assert abs(pipeline.high_step_constants(32760)[0] - 0.8421916) < 1e-7  # P:528 "0.84"


@pytest.mark.parametrize("n,bq,bk", [(250, 64, 16), (300, 128, 80), (130, 32, 48)])
def test_rect_block_energy_against_materialised_P(orc, n, bq, bk):
    """E on a B_q x B_kv grid (P:495-507 with P:1294-1328) = block sums of the materialised
    dense P / |I_r|; rows sum to 1; summing the 16-wide columns of a refined grid gives E."""
    q, k, _ = _rand(n, 16, 4)
    P = scipy.special.softmax(0.25 * (q @ k.T), axis=1)
    E = orc.block_energy(q, k, 0.25, bq, block_kv=bk)
    rb, cb = _block_of(n, bq), _block_of(n, bk)
    ref = np.zeros_like(E)
    np.add.at(ref, (rb[:, None].repeat(n, 1), cb[None, :].repeat(n, 0)), P)
    ref /= np.bincount(rb)[:, None]
    assert np.max(np.abs(E - ref)) < 1e-12 and np.allclose(E.sum(axis=1), 1.0, atol=1e-12)
    fine = orc.block_energy(q, k, 0.25, bq, block_kv=16)
    coarse = np.zeros_like(E)
    np.add.at(coarse, (slice(None), (np.arange(fine.shape[1]) * 16) // bk), fine)
    assert np.max(np.abs(coarse - E)) < 1e-12
