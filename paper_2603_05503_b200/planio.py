"""Plan dictionary and calibration state on disk (checkpoint / resume).

The paper computes the masks once and preloads them at inference; its memory footprint
is the stated limitation.  Two versioned, checksummed binary formats, written
and read here as plain byte layouts (no arithmetic of the method):

  CSAP v1  a compiled plan (csa_plan_t of include/csa.h): header + the ten arrays
  CSAC v1  calibration state: uint16 keep counts, fp64 similarity sums, prompts accumulated --
           written after each prompt so a calibration run can resume where it stopped

Layout of both: magic (4 B) | version u32 | header length u32 | header (little-endian fields,
see _HDR_*) | arrays back to back, each preceded by its byte length (u64) | CRC32 (u32) of
everything before it.  Loading checks magic, version, every length against the header's
geometry and the checksum, and raises ValueError on any mismatch (a truncated or corrupted file
never yields a plan); load_plan then runs csa_validate_plan on the device copy.
"""
from __future__ import annotations

import struct
import zlib

import numpy as np
import torch

from .inputs import Layout

_MAGIC_PLAN = b"CSAP"
_MAGIC_CAL = b"CSAC"
_VERSION = 1
# layout F, H, W, B, B_kv (int32 x 5), n_cells (int64), blk entries (int64), intervals (int64)
_HDR_PLAN = struct.Struct("<5iqqq")
# layout (int32 x 5), n_cells (int64), prompts (int64)
_HDR_CAL = struct.Struct("<5iqq")
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
    blob = bytearray(magic + struct.pack("<II", _VERSION, len(header)) + header)
    for a in arrays:
        raw = np.ascontiguousarray(a).tobytes()
        blob += struct.pack("<Q", len(raw)) + raw
    blob += struct.pack("<I", zlib.crc32(bytes(blob)) & 0xFFFFFFFF)
    with open(path, "wb") as fh:
        fh.write(bytes(blob))


def _read(path: str, magic: bytes, hdr: struct.Struct):
    with open(path, "rb") as fh:
        blob = fh.read()
    if len(blob) < 16 or blob[:4] != magic:
        raise ValueError(f"{path}: not a {magic.decode()} file")
    (crc,) = struct.unpack_from("<I", blob, len(blob) - 4)
    if zlib.crc32(blob[:-4]) & 0xFFFFFFFF != crc:
        raise ValueError(f"{path}: checksum mismatch (corrupted or truncated)")
    version, hlen = struct.unpack_from("<II", blob, 4)
    if version != _VERSION or hlen != hdr.size:
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
        t = torch.from_numpy(a.view(np.int16) if dt == np.uint16 else a.copy())
        t = t.to(device)
        out[name] = t.view(torch.uint16) if dt == np.uint16 else t
    plan = csa.Plan(lay, n_cells, **out)
    plan.kind_host = out["kind"].cpu().tolist()
    plan.anchor_k_host = out["anchor_k"].cpu().tolist()
    if validate and torch.device(device).type == "cuda":
        csa.validate_plan(plan)
    return plan


def save_calibration(path: str, lay: Layout, keep_count: torch.Tensor, sim_sum: torch.Tensor,
                     prompts: int) -> None:
    """Calibration state after `prompts` prompts: keep counts uint16 [cells, N_B, N_Bkv] and the
    fp64 similarity sums [cells] (csa_calib_accumulate / csa_spatial_similarity accumulators)."""
    cells = sim_sum.numel()
    if keep_count.numel() != cells * lay.NB * lay.NBK:
        raise ValueError("keep_count does not match the layout and cell count")
    header = _HDR_CAL.pack(lay.F, lay.H, lay.W, lay.B, lay.BK, cells, prompts)
    _write(path, _MAGIC_CAL, header, [_host(keep_count.reshape(-1), np.uint16),
                                      _host(sim_sum, np.float64)])


def load_calibration(path: str, device="cuda"):
    """-> (layout, keep_count uint16 [cells * N_B * N_Bkv], sim_sum fp64 [cells], prompts),
    ready to pass back to csa.calib_accumulate / csa.spatial_similarity to continue."""
    (F, H, W, B, BK, cells, prompts), raw = _read(path, _MAGIC_CAL, _HDR_CAL)
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
