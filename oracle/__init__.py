"""fp64 CPU oracle for the calibrated-sparse-attention hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2603_05503_b200``) never imports it; the two share no code.

Thin ctypes marshalling around ``csa_oracle.c`` (plain C, fp64, ``-ffp-contract=off``).
Each wrapper names the PAPER.md passage its C function writes out; see the C file header for
the readings (Q1..Q22) of passages the paper leaves open.

Parity status: every function here is pinned by ``tests/test_oracle_*.py`` (brute force, closed
forms, paper-printed values).  There is no "parity unpinned" function in this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csa_oracle.c")
_LIB = os.path.join(_HERE, "libcsa_oracle.so")

_c_i32 = ctypes.c_int32
_c_i64 = ctypes.c_int64
_c_dbl = ctypes.c_double
_p = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no BLAS, no FMA contraction).  Returns the .so path."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"]
        )
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        L = _lib
        L.csao_num_blocks.restype = _c_i64
        L.csao_num_blocks.argtypes = [_c_i64, _c_i64]
        L.csao_token_index.restype = _c_i64
        L.csao_token_index.argtypes = [_c_i64] * 5
        L.csao_A_of_N.restype = _c_dbl
        L.csao_A_of_N.argtypes = [_c_dbl]
        L.csao_epsilon.restype = _c_dbl
        L.csao_epsilon.argtypes = [_c_i32, _c_i32, _c_dbl, _c_dbl, _c_dbl]
        L.csao_masked_attention_rows.restype = ctypes.c_int
        L.csao_masked_attention_rows.argtypes = [_c_i64, _c_i32, _c_i32, _p, _p, _p, _c_dbl, _p,
                                                 _c_i64, _c_i64, _p, _p]
        L.csao_masked_attention_rows_rect.restype = ctypes.c_int
        L.csao_masked_attention_rows_rect.argtypes = [_c_i64, _c_i32, _c_i32, _c_i32, _p, _p, _p,
                                                      _c_dbl, _p, _c_i64, _c_i64, _p, _p]
        L.csao_compile_cell_rect.restype = ctypes.c_int
        L.csao_compile_cell_rect.argtypes = [_c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _c_i32, _p,
                                             _c_i32, _c_i32, _c_dbl, _c_dbl, _c_i32, _p, _p, _p,
                                             _p, _p, _p, _p]
        L.csao_anchor_rows.restype = ctypes.c_int
        L.csao_anchor_rows.argtypes = [_c_i32, _c_i32, _p]
        L.csao_nearest_anchor.restype = _c_i32
        L.csao_nearest_anchor.argtypes = [_c_i32, _c_i32, _c_i32]
        L.csao_anchor_attention_rows.restype = ctypes.c_int
        L.csao_anchor_attention_rows.argtypes = [_c_i32, _c_i32, _c_i32, _c_i32, _p, _p, _p,
                                                 _c_dbl, _c_i32, _c_i64, _c_i64, _p, _p]
        L.csao_spatial_cos.restype = ctypes.c_int
        L.csao_spatial_cos.argtypes = [_c_i32, _c_i32, _c_i32, _c_i32, _p, _p, _c_dbl, _c_i32,
                                       _c_i32, _c_i32, _p]
        L.csao_percentile_nearest_rank.restype = _c_i32
        L.csao_percentile_nearest_rank.argtypes = [_c_i64, _p, _c_dbl]
        L.csao_merge_row.restype = _c_i32
        L.csao_merge_row.argtypes = [_c_i32, _p, _c_i32, _p]
        L.csao_skipped_iou.restype = _c_dbl
        L.csao_skipped_iou.argtypes = [_c_i64, _p, _p]
        L.csao_cluster_timesteps.restype = _c_i32
        L.csao_cluster_timesteps.argtypes = [_c_i32, _p, _c_dbl, _p]
        L.csao_row_lse.restype = ctypes.c_int
        L.csao_row_lse.argtypes = [_c_i64, _c_i32, _p, _p, _c_dbl, _c_i64, _c_i64, _p]
        L.csao_block_energy_rows.restype = ctypes.c_int
        L.csao_block_energy_rows.argtypes = [_c_i64, _c_i32, _c_i32, _p, _p, _c_dbl, _p,
                                             _c_i64, _c_i64, _p]
        L.csao_block_energy_rows_rect.restype = ctypes.c_int
        L.csao_block_energy_rows_rect.argtypes = [_c_i64, _c_i32, _c_i32, _c_i32, _p, _p, _c_dbl,
                                                  _p, _c_i64, _c_i64, _p]
        L.csao_select.restype = _c_i32
        L.csao_select.argtypes = [_c_i32, _p, _c_dbl, _p]
        L.csao_accumulate.restype = None
        L.csao_accumulate.argtypes = [_c_i64, _p, _p]
        L.csao_min_count.restype = _c_i32
        L.csao_min_count.argtypes = [_c_dbl, _c_i32]
        L.csao_compile_cell.restype = ctypes.c_int
        L.csao_compile_cell.argtypes = [_c_i64, _c_i32, _c_i32, _c_i32, _c_i32, _p, _c_i32, _c_i32,
                                        _c_dbl, _c_dbl, _c_i32, _p, _p, _p, _p, _p, _p, _p]
        L.csao_work_list.restype = _c_i64
        L.csao_work_list.argtypes = [_c_i32, _c_i64, _c_i32, _c_i32, _c_i32, _p, _p, _p, _c_i32, _p,
                                     _c_i64]
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def num_blocks(n: int, b: int) -> int:
    """N_B = ceil(N/B) (P:196-204 Eq. eq:indices, ragged-aware, Q2)."""
    return int(lib().csao_num_blocks(n, b))


def token_index(H: int, W: int, f: int, i: int, j: int) -> int:
    """Row-major token index f*H*W + i*W + j."""
    return int(lib().csao_token_index(H, W, f, i, j))


def A_of_N(n: float) -> float:
    """A(N) = 0.796 + 1.41e-6 N."""
    return float(lib().csao_A_of_N(float(n)))


def epsilon(t: int, T: int, A: float, C: float, k: float) -> float:
    """eps(t) = A + (C-A) exp(-k t/T) (Eq. eq:epsilon_schedule)."""
    return float(lib().csao_epsilon(t, T, A, C, k))


def masked_attention_rows(q, k, v, scale: float, block: int, mask=None, rows=None,
                          block_kv: int | None = None):
    """Masked-softmax attention of one head (Q1, Q2).

    q, k, v: [N, d]; mask: [N_B, N_Bkv] {0,1} or None (dense); rows: (begin, end) token range;
    block_kv: key block size B_kv of non-square B_q x B_kv blocks, None -> block.
    Returns (out [rows, d] float64, lse [rows] float64, natural log).
    """
    q, k, v = _f64(q), _f64(k), _f64(v)
    n, d = q.shape
    r0, r1 = (0, n) if rows is None else rows
    out = np.empty((r1 - r0, d), np.float64)
    lse = np.empty((r1 - r0,), np.float64)
    m = None if mask is None else np.ascontiguousarray(np.asarray(mask, dtype=np.uint8))
    bk = block if block_kv is None else block_kv
    rc = lib().csao_masked_attention_rows_rect(n, d, block, bk, _ptr(q), _ptr(k), _ptr(v), scale,
                                               None if m is None else _ptr(m), r0, r1, _ptr(out),
                                               _ptr(lse))
    if rc != 0:
        raise ValueError("csao_masked_attention_rows: invalid argument")
    return out, lse


def anchor_rows(H: int, k: int) -> list[int]:
    """a_m = floor((2m+1)H/(2k)) (P:616-622 'equispaced', reading Q9)."""
    out = np.empty((k,), np.int32)
    if lib().csao_anchor_rows(H, k, _ptr(out)) != 0:
        raise ValueError("anchor_rows: need 1 <= k <= H")
    return [int(x) for x in out]


def nearest_anchor(H: int, k: int, i: int) -> int:
    """Index m of the anchor nearest to spatial row i (tie -> lower m, Q9)."""
    return int(lib().csao_nearest_anchor(H, k, i))


def anchor_attention_rows(F, H, W, q, k, v, scale: float, kA: int, rows=None):
    """REPETITIVE head output rows (Q10, Q11).  Returns (out, lse)."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    n, d = q.shape
    assert n == F * H * W
    r0, r1 = (0, n) if rows is None else rows
    out = np.empty((r1 - r0, d), np.float64)
    lse = np.empty((r1 - r0,), np.float64)
    rc = lib().csao_anchor_attention_rows(F, H, W, d, _ptr(q), _ptr(k), _ptr(v), scale, kA, r0, r1,
                                          _ptr(out), _ptr(lse))
    if rc != 0:
        raise ValueError("csao_anchor_attention_rows: invalid argument")
    return out, lse


def spatial_cos(F, H, W, q, k, scale: float, kA: int, f: int, i: int) -> float:
    """cos(P^(f,i), P^(f,a(i))) of one prompt (readings Q23-Q25): flattened W x N
    blocks of the dense map, query (f,i,j) paired with (f,a(i),j)."""
    q, k = _f64(q), _f64(k)
    n, d = q.shape
    assert n == F * H * W
    out = np.empty((1,), np.float64)
    if lib().csao_spatial_cos(F, H, W, d, _ptr(q), _ptr(k), scale, kA, f, i, _ptr(out)) != 0:
        raise ValueError("spatial_cos: invalid argument")
    return float(out[0])


def spatial_similarity(F, H, W, q, k, scale: float, kA: int) -> float:
    """s of one prompt: mean of spatial_cos over every (f, i) (reading Q24)."""
    return float(np.mean([spatial_cos(F, H, W, q, k, scale, kA, f, i)
                          for f in range(F) for i in range(H)]))


def percentile_nearest_rank(values, p: float) -> int:
    """Nearest-rank p-th percentile (sorted ascending, element ceil(p/100 n)); reading Q26."""
    v = np.ascontiguousarray(values, dtype=np.int32)
    out = lib().csao_percentile_nearest_rank(v.size, _ptr(v), float(p))
    if out < 0:
        raise ValueError("percentile: need n > 0 and 0 < p <= 100")
    return int(out)


def merge_row(intervals, target: int):
    """Greedy smallest-gap (leftmost) merging of one row's intervals until count <= target
    (reading Q28).  Returns (merged [(s, e), ...], added blocks)."""
    iv = np.ascontiguousarray(np.asarray(intervals, dtype=np.uint16).reshape(-1, 2))
    added = np.zeros(1, np.int64)
    n = lib().csao_merge_row(iv.shape[0], _ptr(iv), int(target), _ptr(added))
    return [tuple(int(x) for x in iv[i]) for i in range(n)], int(added[0])


def skipped_iou(kept1, kept2) -> float:
    """|S1 & S2| / |S1 | S2| over skipped blocks (Eq. eq:timestep_iou); 1 if both empty."""
    a = np.ascontiguousarray(kept1, dtype=np.uint8).ravel()
    b = np.ascontiguousarray(kept2, dtype=np.uint8).ravel()
    assert a.size == b.size
    return float(lib().csao_skipped_iou(a.size, _ptr(a), _ptr(b)))


def cluster_timesteps(iou, tau: float):
    """Greedy cliques over timesteps (reading Q27).  Returns cluster ids [T]."""
    m = np.ascontiguousarray(iou, dtype=np.float64)
    T = m.shape[0]
    out = np.empty(T, np.int32)
    lib().csao_cluster_timesteps(T, _ptr(m), float(tau), _ptr(out))
    return out


def row_lse(q, k, scale: float, rows=None) -> np.ndarray:
    """lse_i over all N keys of the dense map, natural log."""
    q, k = _f64(q), _f64(k)
    n, d = q.shape
    r0, r1 = (0, n) if rows is None else rows
    out = np.empty((r1 - r0,), np.float64)
    if lib().csao_row_lse(n, d, _ptr(q), _ptr(k), scale, r0, r1, _ptr(out)) != 0:
        raise ValueError("row_lse: invalid argument")
    return out


def block_energy(q, k, scale: float, block: int, lse=None, block_rows=None,
                 block_kv: int | None = None) -> np.ndarray:
    """E_{r,c} (Eq. eq:block_energy; divides by |I_r|, Q2).  Returns [rows, N_Bkv];
    block_kv: key block size of non-square B_q x B_kv blocks, None -> block."""
    q, k = _f64(q), _f64(k)
    n, d = q.shape
    bk = block if block_kv is None else block_kv
    nb = num_blocks(n, bk)
    r0, r1 = (0, num_blocks(n, block)) if block_rows is None else block_rows
    out = np.empty((r1 - r0, nb), np.float64)
    l = None if lse is None else _f64(lse)
    rc = lib().csao_block_energy_rows_rect(n, d, block, bk, _ptr(q), _ptr(k), scale,
                                           None if l is None else _ptr(l), r0, r1, _ptr(out))
    if rc != 0:
        raise ValueError("block_energy: invalid argument")
    return out


def select(E_row, eps: float) -> np.ndarray:
    """Shortest prefix of (E desc, c asc) with fp64 sequential sum >= eps (
    Q4, Q5).  Returns a {0,1} uint8 vector."""
    e = _f64(E_row)
    kept = np.zeros(e.shape[0], np.uint8)
    if lib().csao_select(e.shape[0], _ptr(e), eps, _ptr(kept)) < 0:
        raise MemoryError("select")
    return kept


def accumulate(kept, count: np.ndarray) -> None:
    """count += kept in place (Eq. eq:mask_mean numerator); uint16 saturating."""
    kk = np.ascontiguousarray(np.asarray(kept, dtype=np.uint8))
    assert count.dtype == np.uint16 and count.flags.c_contiguous and count.size == kk.size
    lib().csao_accumulate(kk.size, _ptr(kk), _ptr(count))


def min_count(rho: float, n_prompts: int) -> int:
    """Smallest integer c with c >= rho*|D| (Eq. eq:mask_threshold in count space, Q6)."""
    return int(lib().csao_min_count(rho, n_prompts))


def compile_cell(count, n: int, block: int, F: int, H: int, W: int, min_count_: int,
                 similarity=None, gamma: float = 0.87, anchor_k: int = 5,
                 block_kv: int | None = None) -> dict:
    """Plan for one cell (Q6-Q8); block_kv: key block
    size of non-square B_q x B_kv blocks: count / mask are [N_B, N_Bkv]."""
    nbq = num_blocks(n, block)
    bk = block if block_kv is None else block_kv
    nb = num_blocks(n, bk)
    cnt = np.ascontiguousarray(np.asarray(count, dtype=np.uint16).reshape(nbq, nb))
    kind = np.zeros(1, np.uint8)
    mask = np.zeros((nbq, nb), np.uint8)
    brp = np.zeros(nbq + 1, np.int32)
    bidx = np.zeros(nbq * nb, np.uint16)
    irp = np.zeros(nbq + 1, np.int32)
    ivl = np.zeros(2 * nbq * nb, np.uint16)
    area = np.zeros(1, np.int64)
    rc = lib().csao_compile_cell_rect(n, block, bk, F, H, W, _ptr(cnt), min_count_,
                                 0 if similarity is None else 1,
                                 0.0 if similarity is None else float(similarity), gamma, anchor_k,
                                 _ptr(kind), _ptr(mask), _ptr(brp), _ptr(bidx), _ptr(irp),
                                 _ptr(ivl), _ptr(area))
    if rc != 0:
        raise ValueError("compile_cell: invalid argument")
    return {
        "kind": int(kind[0]),
        "mask": mask,
        "blk_row_ptr": brp,
        "blk_idx": bidx[: brp[-1]].copy(),
        "ivl_row_ptr": irp,
        "ivl": ivl[: 2 * irp[-1]].reshape(-1, 2).copy(),
        "kept_area": int(area[0]),
    }


def work_list(n: int, block: int, F: int, W: int, kinds, anchor_k, row_nnz, order: int = 0
              ) -> np.ndarray:
    """Work list of one launch (scheduling artefact): order 0 longest-first,
    1 natural, 2 head-major longest-first within a head, 3 the same over pair items (2p, 2p+1)."""
    kinds = np.ascontiguousarray(np.asarray(kinds, dtype=np.uint8))
    ak = np.ascontiguousarray(np.asarray(anchor_k, dtype=np.int32))
    nnz = np.ascontiguousarray(np.asarray(row_nnz, dtype=np.int32))
    nb = num_blocks(n, block)
    cap = int(kinds.size * max(nb, (F * int(ak.max(initial=1)) * W + 127) // 128) + 1)
    out = np.zeros(cap, np.uint32)
    cnt = lib().csao_work_list(kinds.size, n, block, F, W, _ptr(kinds), _ptr(ak), _ptr(nnz),
                               order, _ptr(out), cap)
    if cnt < 0:
        raise ValueError("work_list: capacity")
    return out[:cnt].copy()


def sparsity_of_cell(kept_area: int, n: int) -> float:
    """Fraction of skipped query-key pairs of one cell: 1 - kept_area / N^2."""
    return 1.0 - float(kept_area) / float(n * n)
