"""Python binding of libcsa.so (include/csa.h): argument marshalling only.

Every step of the hot path runs in the CUDA kernels behind the C ABI; this module only turns
torch tensors into pointers/strides and owns the plan buffers' allocation (torch, device memory).
There is no CPU fallback: importing this module without a built libcsa.so raises, and every call
needs CUDA tensors on an sm_100 device.
"""
from __future__ import annotations

import ctypes
import dataclasses
import math
import os

import torch

from .inputs import Layout

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CSA_LIB") or os.path.join(_HERE, "libcsa.so")  # CSA_LIB: A/B builds

CSA_OK = 0
_STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "UNSUPPORTED", 3: "CORRUPT_PLAN", 4: "CUDA",
           5: "INSUFFICIENT_CAPACITY"}


class CsaError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where}: CSA_{_STATUS.get(status, status)}: {detail}")
        self.status = status


class _LayoutT(ctypes.Structure):
    _fields_ = [("frames", ctypes.c_int32), ("rows", ctypes.c_int32), ("cols", ctypes.c_int32),
                ("block", ctypes.c_int32), ("block_kv", ctypes.c_int32)]


class _TensorT(ctypes.Structure):
    _fields_ = [("ptr", ctypes.c_void_p), ("stride_b", ctypes.c_int64),
                ("stride_n", ctypes.c_int64), ("stride_h", ctypes.c_int64)]


class _PlanT(ctypes.Structure):
    _fields_ = [("n_cells", ctypes.c_int64), ("kind", ctypes.c_void_p),
                ("anchor_k", ctypes.c_void_p), ("mask_bits", ctypes.c_void_p),
                ("blk_base", ctypes.c_void_p), ("blk_row_ptr", ctypes.c_void_p),
                ("blk_idx", ctypes.c_void_p), ("ivl_base", ctypes.c_void_p),
                ("ivl_row_ptr", ctypes.c_void_p), ("ivl", ctypes.c_void_p),
                ("kept_area", ctypes.c_void_p), ("blk_capacity", ctypes.c_int64),
                ("ivl_capacity", ctypes.c_int64)]


EXPORTS = ["csa_calib_accumulate", "csa_compile_plan", "csa_build_work_list",
           "csa_sparse_attn_fwd", "csa_workspace_size", "csa_validate_plan", "csa_last_error",
           "csa_version", "csa_debug_trace", "csa_spatial_similarity", "csa_merge_intervals",
           "csa_share_timesteps", "csa_copy_heads", "csa_calib_accumulate_sim",
           "csa_sparse_attn_fwd_scatter"]

_lib = None


def lib() -> ctypes.CDLL:
    """Load libcsa.so (fails loudly if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (nvcc, sm_100a).  There is no CPU fallback.")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, st = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int
    L.csa_last_error.restype = ctypes.c_char_p
    L.csa_version.restype = ctypes.c_char_p
    L.csa_workspace_size.restype = ctypes.c_size_t
    L.csa_workspace_size.argtypes = [i32, _LayoutT, i32, i32]
    L.csa_calib_accumulate.restype = st
    L.csa_calib_accumulate.argtypes = [_LayoutT, i32, i32, ctypes.c_float, _TensorT, _TensorT, vp,
                                       ctypes.c_double, vp, vp, vp, vp, ctypes.c_size_t, vp]
    L.csa_calib_accumulate_sim.restype = st
    L.csa_calib_accumulate_sim.argtypes = [_LayoutT, i32, i32, ctypes.c_float, _TensorT, _TensorT,
                                           ctypes.c_double, vp, vp, vp, i32, vp, vp, vp,
                                           ctypes.c_size_t, vp]
    L.csa_compile_plan.restype = st
    L.csa_compile_plan.argtypes = [_LayoutT, i64, vp, i32, vp, ctypes.c_double, i32, i32,
                                   ctypes.POINTER(_PlanT), vp, ctypes.c_size_t, vp]
    L.csa_build_work_list.restype = st
    L.csa_build_work_list.argtypes = [_LayoutT, ctypes.POINTER(_PlanT), i64, i32, i32, vp, i32, vp,
                                      vp, ctypes.c_size_t, vp]
    L.csa_sparse_attn_fwd.restype = st
    L.csa_sparse_attn_fwd.argtypes = [_LayoutT, i32, i32, i32, ctypes.c_float, _TensorT, _TensorT,
                                      _TensorT, _TensorT, vp, ctypes.POINTER(_PlanT), i64, vp, vp,
                                      i32, i32, vp, ctypes.c_size_t, vp]
    L.csa_sparse_attn_fwd_scatter.restype = st
    L.csa_sparse_attn_fwd_scatter.argtypes = [_LayoutT, i32, i32, i32, ctypes.c_float, _TensorT,
                                              _TensorT, _TensorT, vp, i32, i64, i64, i64, vp,
                                              ctypes.POINTER(_PlanT), i64, vp, vp, i32, vp,
                                              ctypes.c_size_t, vp]
    L.csa_spatial_similarity.restype = st
    L.csa_spatial_similarity.argtypes = [_LayoutT, i32, i32, ctypes.c_float, _TensorT, _TensorT,
                                         vp, i32, vp, vp, vp, ctypes.c_size_t, vp]
    L.csa_merge_intervals.restype = st
    L.csa_merge_intervals.argtypes = [_LayoutT, i64, ctypes.POINTER(_PlanT), ctypes.c_double, i32,
                                      vp, vp, vp, vp, ctypes.c_size_t, vp]
    L.csa_share_timesteps.restype = st
    L.csa_share_timesteps.argtypes = [_LayoutT, i32, i32, ctypes.POINTER(_PlanT), ctypes.c_double,
                                      i32, vp, vp, vp, vp]
    L.csa_copy_heads.restype = st
    L.csa_copy_heads.argtypes = [vp, vp, _LayoutT, i32, i32, i32, i32, i32, vp]
    L.csa_debug_trace.restype = st
    L.csa_debug_trace.argtypes = [vp, i32]
    L.csa_validate_plan.restype = st
    L.csa_validate_plan.argtypes = [ctypes.POINTER(_PlanT), _LayoutT, i64, vp]
    _lib = L
    return L


def _check(status: int, where: str) -> None:
    if status != CSA_OK:
        raise CsaError(status, where, lib().csa_last_error().decode())


def _layout(lay: Layout) -> _LayoutT:
    return _LayoutT(lay.F, lay.H, lay.W, lay.B, lay.BK)


def _tensor(t: torch.Tensor | None) -> _TensorT:
    if t is None:
        return _TensorT(None, 0, 0, 0)
    if t.dtype != torch.bfloat16 or not t.is_cuda or t.dim() != 4 or t.stride(3) != 1:
        raise ValueError("expected a CUDA bf16 tensor [batch, N, heads, head_dim], head_dim "
                         "contiguous")
    return _TensorT(t.data_ptr(), t.stride(0), t.stride(1), t.stride(2))


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def default_scale(d: int) -> float:
    """softmax scale 1/sqrt(d)."""
    return 1.0 / math.sqrt(d)


# ------------------------------------------------------------------------------- calibration
def calib_accumulate(lay: Layout, q: torch.Tensor, k: torch.Tensor, eps: float,
                     keep_count: torch.Tensor, lse_in: torch.Tensor | None = None,
                     energy_out: torch.Tensor | None = None, lse_out: torch.Tensor | None = None,
                     scale: float | None = None, stream=None, single_pass: bool = True) -> None:
    """csa_calib_accumulate: one prompt at one (t, l), all heads of q/k [1, N, H, d].
    single_pass: hand the kernel its scratch workspace (one exponential pass when lse_in is
    None); False -> the two-pass path."""
    _, n, heads, d = q.shape
    assert n == lay.N and keep_count.dtype == torch.uint16 and keep_count.is_contiguous()
    assert keep_count.numel() == heads * lay.NB * lay.NBK
    for t, shape in ((lse_in, heads * n), (lse_out, heads * n),
                     (energy_out, heads * lay.NB * lay.NBK)):
        if t is not None:
            assert t.dtype == torch.float32 and t.is_contiguous() and t.numel() == shape
    sc = default_scale(d) if scale is None else scale
    ws, ws_bytes = None, 0
    if single_pass and lse_in is None:
        ws_bytes = lib().csa_workspace_size(0, _layout(lay), heads, d)
        ws = _calib_workspace(q.device, ws_bytes)
    _check(lib().csa_calib_accumulate(_layout(lay), heads, d, sc, _tensor(q), _tensor(k),
                                      _ptr(lse_in), float(eps), _ptr(keep_count),
                                      _ptr(energy_out), _ptr(lse_out), _ptr(ws), ws_bytes,
                                      _stream(stream)),
           "csa_calib_accumulate")


def calib_accumulate_sim(lay: Layout, q: torch.Tensor, k: torch.Tensor, eps: float,
                         keep_count: torch.Tensor, anchor_k: int, sim_sum: torch.Tensor,
                         energy_out: torch.Tensor | None = None,
                         lse_out: torch.Tensor | None = None, cos_out: torch.Tensor | None = None,
                         scale: float | None = None, stream=None) -> None:
    """csa_calib_accumulate_sim: calib_accumulate (a2-a5) and spatial_similarity (f1) of one
    prompt in one pass over the key tiles."""
    _, n, heads, d = q.shape
    assert n == lay.N and keep_count.dtype == torch.uint16 and keep_count.is_contiguous()
    assert keep_count.numel() == heads * lay.NB * lay.NBK
    assert sim_sum.dtype == torch.float64 and sim_sum.numel() == heads
    for t, shape in ((lse_out, heads * n), (energy_out, heads * lay.NB * lay.NBK),
                     (cos_out, heads * lay.F * lay.H)):
        if t is not None:
            assert t.dtype == torch.float32 and t.is_contiguous() and t.numel() == shape
    sc = default_scale(d) if scale is None else scale
    nbytes = lib().csa_workspace_size(6, _layout(lay), heads, d)
    ws = _calib_workspace(q.device, nbytes, key="calib_sim")
    _check(lib().csa_calib_accumulate_sim(_layout(lay), heads, d, sc, _tensor(q), _tensor(k),
                                          float(eps), _ptr(keep_count), _ptr(energy_out),
                                          _ptr(lse_out), int(anchor_k), _ptr(sim_sum),
                                          _ptr(cos_out), _ptr(ws), nbytes, _stream(stream)),
           "csa_calib_accumulate_sim")


def spatial_similarity(lay: Layout, q: torch.Tensor, k: torch.Tensor, lse: torch.Tensor,
                       anchor_k: int, sim_sum: torch.Tensor, cos_out: torch.Tensor | None = None,
                       scale: float | None = None, stream=None) -> None:
    """csa_spatial_similarity (f1): sim_sum[h] += sum over (f, i) of
    cos(P^(f,i), P^(f,a(i))) for one prompt; lse [heads * N] fp32 natural log (e.g. the
    calibration pass's lse_out).  s[h] = sim_sum[h] / (F * H * prompts) feeds compile_plan."""
    _, n, heads, d = q.shape
    assert n == lay.N and lse.dtype == torch.float32 and lse.numel() == heads * n
    assert sim_sum.dtype == torch.float64 and sim_sum.numel() == heads
    if cos_out is not None:
        assert cos_out.dtype == torch.float32 and cos_out.numel() == heads * lay.F * lay.H
    sc = default_scale(d) if scale is None else scale
    nbytes = lib().csa_workspace_size(4, _layout(lay), heads, d)
    ws = _calib_workspace(q.device, nbytes, key="sim")
    _check(lib().csa_spatial_similarity(_layout(lay), heads, d, sc, _tensor(q), _tensor(k),
                                        _ptr(lse), int(anchor_k), _ptr(sim_sum), _ptr(cos_out),
                                        _ptr(ws), nbytes, _stream(stream)),
           "csa_spatial_similarity")


_CALIB_WS: dict = {}


def _calib_workspace(device, nbytes: int, key: str = "calib") -> torch.Tensor:
    """Cached scratch for the single-pass calibration / the similarity pass (grown on demand),
    one per (device, current stream, use): calls on one stream are ordered, so they can share
    it; calls on different streams never do.  A replaced buffer is kept alive (a captured CUDA
    graph may still hold its address)."""
    s = torch.cuda.current_stream(device)
    key = (key, torch.device(device).index, s.cuda_stream)
    buf = _CALIB_WS.get(key)
    if buf is None or buf.numel() < nbytes:
        if buf is not None:
            _RETIRED_WS.append(buf)
        buf = torch.empty(max(nbytes, 16), dtype=torch.uint8, device=device)
        _CALIB_WS[key] = buf
    return buf


# ------------------------------------------------------------------------------- plan
@dataclasses.dataclass
class Plan:
    """Device buffers of a compiled plan (see csa_plan_t in include/csa.h)."""

    lay: Layout
    n_cells: int
    kind: torch.Tensor
    anchor_k: torch.Tensor
    mask_bits: torch.Tensor
    blk_base: torch.Tensor
    blk_row_ptr: torch.Tensor
    blk_idx: torch.Tensor
    ivl_base: torch.Tensor
    ivl_row_ptr: torch.Tensor
    ivl: torch.Tensor
    kept_area: torch.Tensor
    kind_host: list | None = None
    anchor_k_host: list | None = None

    def struct(self) -> _PlanT:
        return _PlanT(self.n_cells, self.kind.data_ptr(), self.anchor_k.data_ptr(),
                      self.mask_bits.data_ptr(), self.blk_base.data_ptr(),
                      self.blk_row_ptr.data_ptr(),
                      self.blk_idx.data_ptr() if self.blk_idx.numel() else None,
                      self.ivl_base.data_ptr(), self.ivl_row_ptr.data_ptr(),
                      self.ivl.data_ptr() if self.ivl.numel() else None,
                      self.kept_area.data_ptr(), self.blk_idx.numel(), self.ivl.numel() // 2)

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in (
            self.kind, self.anchor_k, self.mask_bits, self.blk_base, self.blk_row_ptr,
            self.blk_idx, self.ivl_base, self.ivl_row_ptr, self.ivl, self.kept_area))

    def items(self, cell_base: int, n_heads: int, pairs: bool = False) -> int:
        """Work items of one launch (host-side count used to size the persistent grid)."""
        tot = 0
        for h in range(n_heads):
            c = cell_base + h
            if self.kind_host[c]:
                units = (self.lay.F * self.anchor_k_host[c] * self.lay.W + 127) // 128
            else:
                units = self.lay.NB
            tot += (units + 1) // 2 if pairs else units
        return tot


def compile_plan(lay: Layout, keep_count: torch.Tensor, min_count: int,
                 similarity: torch.Tensor | None = None, gamma: float = 0.87, anchor_k: int = 5,
                 stream=None, csr: bool = True) -> Plan:
    """csa_compile_plan phase 0 (count) -> size read-back -> phase 1 (fill).  csr=False: an
    intervals-only plan (no blk_idx: the kernels walk the 1-D skip list)."""
    dev = keep_count.device
    nb, nbk = lay.NB, lay.NBK
    n_cells = keep_count.numel() // (nb * nbk)
    assert keep_count.dtype == torch.uint16 and keep_count.is_contiguous()
    if similarity is not None:
        assert similarity.dtype == torch.float64 and similarity.numel() == n_cells
    w32 = (nbk + 31) // 32
    e = torch.empty
    p = Plan(lay, n_cells,
             kind=e(n_cells, dtype=torch.uint8, device=dev),
             anchor_k=e(n_cells, dtype=torch.int32, device=dev),
             mask_bits=e(n_cells * nb * w32, dtype=torch.int32, device=dev),
             blk_base=e(n_cells + 1, dtype=torch.int64, device=dev),
             blk_row_ptr=e(n_cells * (nb + 1), dtype=torch.int32, device=dev),
             blk_idx=e(0, dtype=torch.uint16, device=dev),
             ivl_base=e(n_cells + 1, dtype=torch.int64, device=dev),
             ivl_row_ptr=e(n_cells * (nb + 1), dtype=torch.int32, device=dev),
             ivl=e(0, dtype=torch.uint16, device=dev),
             kept_area=e(n_cells, dtype=torch.int64, device=dev))
    s = p.struct()
    _check(lib().csa_compile_plan(_layout(lay), n_cells, _ptr(keep_count), int(min_count),
                                  _ptr(similarity), float(gamma), int(anchor_k), 0,
                                  ctypes.byref(s), None, 0, _stream(stream)), "csa_compile_plan(0)")
    tot_b = int(p.blk_base[n_cells].item())
    tot_i = int(p.ivl_base[n_cells].item())
    p.blk_idx = e(max(tot_b, 1) if csr else 0, dtype=torch.uint16, device=dev)
    p.ivl = e(max(2 * tot_i, 2), dtype=torch.uint16, device=dev)
    s = p.struct()
    _check(lib().csa_compile_plan(_layout(lay), n_cells, None, int(min_count), None, float(gamma),
                                  int(anchor_k), 1, ctypes.byref(s), None, 0, _stream(stream)),
           "csa_compile_plan(1)")
    p.kind_host = p.kind.cpu().tolist()
    p.anchor_k_host = p.anchor_k.cpu().tolist()
    return p


_HOST_BUFS: dict = {}


def sparse_attn_fwd_host(q_h: torch.Tensor, k_h: torch.Tensor, v_h: torch.Tensor, plan: Plan,
                         out_h: torch.Tensor, heads_per_chunk: int = 2,
                         device: torch.device | str = "cuda") -> torch.Tensor:
    """One layer from pinned host Q, K, V [1, N, H, d] to pinned host O, streamed by head chunks:
    H2D of chunk c+1 (csa_copy_heads on a copy stream) overlaps the attention of chunk c (its
    own heads' cells, work list and strided views of the device copies) and the D2H of chunk c-1.
    Device staging buffers and per-chunk work lists are cached.  Returns out_h; synchronous on
    return of the current stream (the caller synchronizes to read out_h)."""
    b, n, heads, d = q_h.shape
    lay = plan.lay
    if b != 1:
        raise ValueError("sparse_attn_fwd_host: batch 1 only (csa_copy_heads moves one sequence)")
    for name, t in (("q", q_h), ("k", k_h), ("v", v_h), ("out", out_h)):
        if t.shape != q_h.shape or t.dtype != torch.bfloat16 or not t.is_pinned() \
                or not t.is_contiguous():
            raise ValueError(f"sparse_attn_fwd_host: {name} must be a pinned, contiguous bf16 "
                             f"tensor of shape {tuple(q_h.shape)} (dense [1, N, H, d] rows)")
    key = (str(device), q_h.shape)
    bufs = _HOST_BUFS.get(key)
    if bufs is None:
        bufs = {"q": torch.empty(q_h.shape, dtype=q_h.dtype, device=device),
                "k": torch.empty(q_h.shape, dtype=q_h.dtype, device=device),
                "v": torch.empty(q_h.shape, dtype=q_h.dtype, device=device),
                "o": torch.empty(q_h.shape, dtype=q_h.dtype, device=device),
                "s_in": torch.cuda.Stream(device=device), "s_out": torch.cuda.Stream(device=device)}
        _HOST_BUFS[key] = bufs
    chunks = [(h0, min(h0 + heads_per_chunk, heads)) for h0 in range(0, heads, heads_per_chunk)]
    wkey = ("chunk_work", heads_per_chunk)
    if getattr(plan, "_chunk_work", None) is None or plan._chunk_work[0] != wkey:
        plan._chunk_work = (wkey, [build_work_list(plan, h0, h1 - h0) for h0, h1 in chunks])
    works = plan._chunk_work[1]
    comp = torch.cuda.current_stream(device)
    s_in, s_out = bufs["s_in"], bufs["s_out"]
    s_in.wait_stream(comp)  # staging buffers free (previous call's reads done)
    for (h0, h1), work in zip(chunks, works):
        for name, src in (("q", q_h), ("k", k_h), ("v", v_h)):
            _check(lib().csa_copy_heads(_ptr(bufs[name]), _ptr(src), _layout(lay), heads, d, h0,
                                        h1, 0, _stream(s_in)), "csa_copy_heads")
        comp.wait_stream(s_in)
        sl = slice(h0, h1)
        sparse_attn_fwd(bufs["q"][:, :, sl], bufs["k"][:, :, sl], bufs["v"][:, :, sl], plan, work,
                        cell_base=h0, out=bufs["o"][:, :, sl], stream=comp)
        s_out.wait_stream(comp)
        _check(lib().csa_copy_heads(_ptr(out_h), _ptr(bufs["o"]), _layout(lay), heads, d, h0, h1,
                                    1, _stream(s_out)), "csa_copy_heads")
    comp.wait_stream(s_out)
    return out_h


def merge_intervals(plan: Plan, keep_count: torch.Tensor, min_count: int, percentile: float,
                    stream=None) -> tuple[torch.Tensor, torch.Tensor]:
    """csa_merge_intervals (f2): fills the smallest gaps of rows wider than the
    nearest-rank `percentile` of the plan's row widths, in keep_count (in place).  Recompile with
    compile_plan(keep_count, min_count) for the merged plan.  Returns device (target, added)."""
    dev = keep_count.device
    assert keep_count.dtype == torch.uint16 and keep_count.is_contiguous()
    target = torch.zeros(1, dtype=torch.int32, device=dev)
    added = torch.zeros(1, dtype=torch.int64, device=dev)
    nbytes = lib().csa_workspace_size(5, _layout(plan.lay), 0, 0)
    ws = torch.empty(max(nbytes, 4), dtype=torch.uint8, device=dev)
    s = plan.struct()
    _check(lib().csa_merge_intervals(_layout(plan.lay), plan.n_cells, ctypes.byref(s),
                                     float(percentile), int(min_count), _ptr(keep_count),
                                     _ptr(target), _ptr(added), _ptr(ws), nbytes, _stream(stream)),
           "csa_merge_intervals")
    return target, added


def share_timesteps(plan: Plan, keep_count: torch.Tensor, n_groups: int, n_steps: int,
                    min_count: int, tau: float, stream=None) -> tuple[torch.Tensor, torch.Tensor]:
    """csa_share_timesteps (f2) over cells (t, g) = t * n_groups + g: skipped-set
    IoU, greedy cliques with IoU >= tau, OR-shared masks written into keep_count (in place).
    Returns device (cluster [n_groups, n_steps] int32, iou [n_groups, n_steps, n_steps] fp64)."""
    dev = keep_count.device
    assert keep_count.dtype == torch.uint16 and keep_count.is_contiguous()
    cluster = torch.empty((n_groups, n_steps), dtype=torch.int32, device=dev)
    iou = torch.empty((n_groups, n_steps, n_steps), dtype=torch.float64, device=dev)
    s = plan.struct()
    _check(lib().csa_share_timesteps(_layout(plan.lay), int(n_groups), int(n_steps),
                                     ctypes.byref(s), float(tau), int(min_count), _ptr(keep_count),
                                     _ptr(cluster), _ptr(iou), _stream(stream)),
           "csa_share_timesteps")
    return cluster, iou


def validate_plan(plan: Plan, n_cells: int | None = None, stream=None) -> None:
    s = plan.struct()
    _check(lib().csa_validate_plan(ctypes.byref(s), _layout(plan.lay),
                                   plan.n_cells if n_cells is None else n_cells, _stream(stream)),
           "csa_validate_plan")


@dataclasses.dataclass
class WorkList:
    items: torch.Tensor   # uint32 codes (stored as int32)
    n_work: torch.Tensor  # device int32 [1]
    max_work: int
    pairs: bool = False   # order 3: items stand for rows (2p, 2p+1) (no kernel in this build)


def default_order(lay: Layout, d: int) -> int:
    """Work-list order of the production path: 2 (head-major, longest row first within a head,
    one CTA per query block at a time)."""
    del lay, d
    return 2


def build_work_list(plan: Plan, cell_base: int, n_heads: int, order: int = 2,
                    stream=None) -> WorkList:
    """csa_build_work_list (orders 0-3, include/csa.h).  order 2: head-major, longest row first
    (the production order)."""
    cap = plan.items(cell_base, n_heads, pairs=(order == 3))
    items = torch.empty(max(cap, 1), dtype=torch.int32, device=plan.kind.device)
    n_work = torch.empty(1, dtype=torch.int32, device=plan.kind.device)
    s = plan.struct()
    _check(lib().csa_build_work_list(_layout(plan.lay), ctypes.byref(s), cell_base, n_heads, order,
                                     _ptr(items), cap, _ptr(n_work), None, 0, _stream(stream)),
           "csa_build_work_list")
    return WorkList(items, n_work, cap, pairs=(order == 3))


# ------------------------------------------------------------------------------- attention
def sparse_attn_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, plan: Plan,
                    work: WorkList, cell_base: int = 0, out: torch.Tensor | None = None,
                    lse_out: torch.Tensor | None = None, scale: float | None = None,
                    stream=None, dynamic: bool = True) -> torch.Tensor:
    """csa_sparse_attn_fwd on q/k/v [batch, N, heads, d] (bf16, CUDA; any token / head stride,
    head_dim contiguous).  dynamic=False: static round-robin item assignment without a workspace
    (block 64 only; block-128 layouts need the workspace for the fallback list, csa.h)."""
    b, n, heads, d = q.shape
    assert n == plan.lay.N and k.shape == q.shape and v.shape == q.shape
    if out is None:
        out = torch.empty_like(q)
    if lse_out is not None:
        assert lse_out.dtype == torch.float32 and lse_out.is_contiguous()
        assert lse_out.numel() == b * heads * n
    sc = default_scale(d) if scale is None else scale
    s = plan.struct()
    ws = _sched_workspace(q.device, lib().csa_workspace_size(3, _layout(plan.lay), heads, d),
                          stream) if dynamic else None
    _check(lib().csa_sparse_attn_fwd(_layout(plan.lay), b, heads, d, sc, _tensor(q), _tensor(k),
                                     _tensor(v), _tensor(out), _ptr(lse_out), ctypes.byref(s),
                                     cell_base, _ptr(work.items), _ptr(work.n_work), work.max_work,
                                     1 if work.pairs else 0, _ptr(ws),
                                     0 if ws is None else ws.numel(), _stream(stream)),
           "csa_sparse_attn_fwd")
    return out


def sparse_attn_fwd_scatter(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, plan: Plan,
                            work: WorkList, peer_ptrs: torch.Tensor, recv_like: torch.Tensor,
                            cell_base: int = 0, lse_out: torch.Tensor | None = None,
                            scale: float | None = None, stream=None) -> None:
    """csa_sparse_attn_fwd_scatter: the attention of q/k/v [batch, N, heads, d] with each output
    row stored into the receive buffer of the rank owning its token: peer_ptrs is a device int64
    tensor [P] of pointers (this rank's first head inside each rank's [batch, N/P, H, d] receive
    buffer), recv_like any tensor with the receive buffers' strides (the Ulysses return exchange
    fused into the epilogue)."""
    b, n, heads, d = q.shape
    assert n == plan.lay.N and k.shape == q.shape and v.shape == q.shape
    assert peer_ptrs.dtype == torch.int64 and peer_ptrs.is_cuda and peer_ptrs.dim() == 1
    if lse_out is not None:
        assert lse_out.dtype == torch.float32 and lse_out.numel() == b * heads * n
    sc = default_scale(d) if scale is None else scale
    s = plan.struct()
    ws = _sched_workspace(q.device, lib().csa_workspace_size(3, _layout(plan.lay), heads, d), stream)
    st_b, st_n, st_h, _ = recv_like.stride()
    _check(lib().csa_sparse_attn_fwd_scatter(_layout(plan.lay), b, heads, d, sc, _tensor(q),
                                             _tensor(k), _tensor(v), _ptr(peer_ptrs),
                                             peer_ptrs.numel(), st_b, st_n, st_h, _ptr(lse_out),
                                             ctypes.byref(s), cell_base, _ptr(work.items),
                                             _ptr(work.n_work), work.max_work, _ptr(ws),
                                             ws.numel(), _stream(stream)),
           "csa_sparse_attn_fwd_scatter")


_SCHED_WS: dict = {}
_RETIRED_WS: list = []


def _sched_workspace(device, nbytes: int, stream=None) -> torch.Tensor:
    """Zero-filled attention workspace (scheduler counters left zero-filled by every launch; the
    fixed-reference kernel's fallback list rewritten by every launch, csa.h), grown on demand,
    one per (device, stream) so launches on different streams never share counters.  A buffer
    replaced by a larger one is kept alive (never freed): a captured CUDA graph may still hold
    its address (stream handles are recycled by torch's stream pool)."""
    s = torch.cuda.current_stream(device) if stream is None else stream
    key = (torch.device(device).index, s.cuda_stream)
    buf = _SCHED_WS.get(key)
    if buf is None or buf.numel() < nbytes:
        if buf is not None:
            _RETIRED_WS.append(buf)
        with torch.cuda.stream(s):
            buf = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        _SCHED_WS[key] = buf
    return buf


def version() -> str:
    return lib().csa_version().decode()
