"""Plan dictionary and calibration state on disk (checkpoint / resume).

The paper computes the masks once and preloads them at inference; its memory footprint
is the stated limitation.  Two versioned, checksummed binary formats, written
and read here as plain byte layouts (no arithmetic of the method):

  CSAP v1  a compiled plan (csa_plan_t of include/csa.h): header + the ten arrays
  CSAC v2  calibration state: uint16 keep counts, fp64 similarity sums, prompts accumulated and
           the settings the counts were accumulated under (dictionary T x L x H, anchor k, rho,
           the eps(t) constants A, C, k of Eq. eq:epsilon_schedule) -- written after each
           prompt so a calibration run can resume where it stopped; resuming under different
           settings is refused instead of silently mixing statistics

Layout of both: magic (4 B) | version u32 | header length u32 | header (little-endian fields,
see _HDR_*) | arrays back to back, each preceded by its byte length (u64) | CRC32 (u32) of
everything before it.  Loading checks magic, version, every length against the header's
geometry and the checksum, and raises ValueError on any mismatch (a truncated or corrupted file
never yields a plan); load_plan then runs csa_validate_plan on the device copy.  Files are
written to `path + ".tmp"`, fsync'ed and renamed over `path`, so a crash mid-write leaves the
previous good file in place.
"""
from __future__ import annotations

import os
import struct
import zlib

import numpy as np
import torch

from .inputs import Layout

_MAGIC_PLAN = b"CSAP"
_MAGIC_CAL = b"CSAC"
_VERSION = {_MAGIC_PLAN: 1, _MAGIC_CAL: 2}
# layout F, H, W, B, B_kv (int32 x 5), n_cells (int64), blk entries (int64), intervals (int64)
_HDR_PLAN = struct.Struct("<5iqqq")
# layout (int32 x 5), n_cells (int64), prompts (int64), T, L, H, anchor k (int32 x 4),
# rho, eps A, eps C, eps k (fp64 x 4)
_HDR_CAL = struct.Struct("<5iqq4i4d")
CAL_SETTINGS = ("T", "L", "H", "anchor_k", "rho", "eps_A", "eps_C", "eps_k")
_PLAN_FIELDS = (("kind", np.uint8), ("anchor_k", np.int32), ("mask_bits", np.int32),
                ("blk_base", np.int64), ("blk_row_ptr", np.int32), ("blk_idx", np.uint16),
                ("ivl_base", np.int64), ("ivl_row_ptr", np.int32), ("ivl", np.uint16),
                ("kept_area", np.int64))


def _host(t: torch.Tensor, dtype) -> np.ndarray:
    """Raw bytes of a (device) tensor as a numpy array of `dtype` (uint16 travels as int16)."""
    if t.dtype == torch.uint16:
        t = t.view(torch.int16)
    return np.ascontiguousarray(t.detach().cpu().numpy()).view(dtype)


def _write(path: str, magic: bytes, header: bytes, arrays) -> None:
    blob = bytearray(magic + struct.pack("<II", _VERSION[magic], len(header)) + header)
    for a in arrays:
        raw = np.ascontiguousarray(a).tobytes()
        blob += struct.pack("<Q", len(raw)) + raw
    blob += struct.pack("<I", zlib.crc32(bytes(blob)) & 0xFFFFFFFF)
    tmp = path + ".tmp"
    with open(tmp, "wb") as fh:
        fh.write(bytes(blob))
        fh.flush()
        os.fsync(fh.fileno())
    os.replace(tmp, path)  # atomic: readers see the old file or the new one, never a torn one


def _read(path: str, magic: bytes, hdr: struct.Struct):
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < 16 or blob[:4] != magic:
        raise ValueError(f"{path}: not a {magic.decode()} file")
    (crc,) = struct.unpack_from("<I", blob, len(blob) - 4)
    if zlib.crc32(blob[:-4]) & 0xFFFFFFFF != crc:
        raise ValueError(f"{path}: checksum mismatch (corrupted or truncated)")
    version, hlen = struct.unpack_from("<II", blob, 4)
    if version != _VERSION[magic] or hlen != hdr.size:
        raise ValueError(f"{path}: unsupported version {version}")
    fields = hdr.unpack_from(blob, 12)
    pos, arrays = 12 + hlen, []
    while pos < len(blob) - 4:
        (n,) = struct.unpack_from("<Q", blob, pos)
        pos += 8
        if pos + n > len(blob) - 4:
            raise ValueError(f"{path}: array overruns the file")
        arrays.append(blob[pos:pos + n])
        pos += n
    return fields, arrays


def save_plan(plan, path: str) -> None:
    """Write a compiled csa.Plan (device or host tensors) as CSAP v1."""
    lay = plan.lay
    arrays = [_host(getattr(plan, name), dt) for name, dt in _PLAN_FIELDS]
    header = _HDR_PLAN.pack(lay.F, lay.H, lay.W, lay.B, lay.BK, plan.n_cells,
                            plan.blk_idx.numel(), plan.ivl.numel() // 2)
    _write(path, _MAGIC_PLAN, header, arrays)


def load_plan(path: str, device="cuda", validate: bool = True):
    """Read a CSAP v1 file into a csa.Plan on `device`; every array length is checked against
    the header's geometry, then (device copies) csa_validate_plan checks the structure."""
    from . import csa

    (F, H, W, B, BK, n_cells, n_blk, n_ivl), raw = _read(path, _MAGIC_PLAN, _HDR_PLAN)
    lay = Layout(F, H, W, B, BK)
    nb, w32 = lay.NB, (lay.NBK + 31) // 32
    expect = {"kind": n_cells, "anchor_k": n_cells, "mask_bits": n_cells * nb * w32,
              "blk_base": n_cells + 1, "blk_row_ptr": n_cells * (nb + 1), "blk_idx": n_blk,
              "ivl_base": n_cells + 1, "ivl_row_ptr": n_cells * (nb + 1), "ivl": 2 * n_ivl,
              "kept_area": n_cells}
    if len(raw) != len(_PLAN_FIELDS):
        raise ValueError(f"{path}: {len(raw)} arrays, expected {len(_PLAN_FIELDS)}")
    out = {}
    for (name, dt), buf in zip(_PLAN_FIELDS, raw):
        a = np.frombuffer(buf, dtype=dt)
        if a.size != expect[name]:
            raise ValueError(f"{path}: {name} has {a.size} entries, expected {expect[name]}")
        t = torch.from_numpy(a.view(np.int16).copy() if dt == np.uint16 else a.copy())
        t = t.to(device)
        out[name] = t.view(torch.uint16) if dt == np.uint16 else t
    plan = csa.Plan(lay, n_cells, **out)
    plan.kind_host = out["kind"].cpu().tolist()
    plan.anchor_k_host = out["anchor_k"].cpu().tolist()
    if validate and torch.device(device).type == "cuda":
        csa.validate_plan(plan)
    return plan


def save_calibration(path: str, lay: Layout, keep_count: torch.Tensor, sim_sum: torch.Tensor,
                     prompts: int, settings: dict | None = None) -> None:
    """Calibration state after `prompts` prompts: keep counts uint16 [cells, N_B, N_Bkv] and the
    fp64 similarity sums [cells] (csa_calib_accumulate / csa_spatial_similarity accumulators),
    with the settings (CAL_SETTINGS keys; missing ones stored as 0) they were accumulated under."""
    cells = sim_sum.numel()
    if keep_count.numel() != cells * lay.NB * lay.NBK:
        raise ValueError("keep_count does not match the layout and cell count")
    st = {k: 0 for k in CAL_SETTINGS}
    st.update(settings or {})
    unknown = set(st) - set(CAL_SETTINGS)
    if unknown:
        raise ValueError(f"unknown calibration settings {sorted(unknown)}")
    header = _HDR_CAL.pack(lay.F, lay.H, lay.W, lay.B, lay.BK, cells, prompts,
                           *(int(st[k]) for k in CAL_SETTINGS[:4]),
                           *(float(st[k]) for k in CAL_SETTINGS[4:]))
    _write(path, _MAGIC_CAL, header, [_host(keep_count.reshape(-1), np.uint16),
                                      _host(sim_sum, np.float64)])


def load_calibration(path: str, device="cuda", expect: dict | None = None):
    """-> (layout, keep_count uint16 [cells * N_B * N_Bkv], sim_sum fp64 [cells], prompts),
    ready to pass back to csa.calib_accumulate / csa.spatial_similarity to continue.  `expect`:
    settings the resumed run uses; any stored value that differs raises ValueError."""
    fields, raw = _read(path, _MAGIC_CAL, _HDR_CAL)
    F, H, W, B, BK, cells, prompts = fields[:7]
    stored = dict(zip(CAL_SETTINGS, fields[7:]))
    for k, v in (expect or {}).items():
        if k not in stored:
            raise ValueError(f"unknown calibration setting {k}")
        if stored[k] != (int(v) if k in CAL_SETTINGS[:4] else float(v)):
            raise ValueError(f"{path}: accumulated with {k} = {stored[k]}, resuming with {v}")
    lay = Layout(F, H, W, B, BK)
    if len(raw) != 2:
        raise ValueError(f"{path}: {len(raw)} arrays, expected 2")
    kc = np.frombuffer(raw[0], dtype=np.uint16)
    ss = np.frombuffer(raw[1], dtype=np.float64)
    if kc.size != cells * lay.NB * lay.NBK or ss.size != cells:
        raise ValueError(f"{path}: array sizes do not match the header")
    keep = torch.from_numpy(kc.view(np.int16).copy()).to(device).view(torch.uint16)
    sim = torch.from_numpy(ss.copy()).to(device)
    return lay, keep, sim, int(prompts)
