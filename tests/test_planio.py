"""Plan / calibration-state files (checkpoint and resume): round trips, corruption and truncation
detection (CPU), and on the GPU a compiled plan that survives save -> load bit for bit."""
import os

import numpy as np
import pytest
import torch

import oracle
from paper_2603_05503_b200 import csa, inputs, planio
from paper_2603_05503_b200.inputs import Layout


def _host_plan(lay, counts, min_count):
    """A csa.Plan assembled on the host from the oracle compiler (test fixture only)."""
    nb, nbk = lay.NB, lay.NBK
    w32 = (nbk + 31) // 32
    cells = [oracle.compile_cell(c, lay.N, lay.B, lay.F, lay.H, lay.W, min_count,
                                 block_kv=lay.BK or None) for c in counts]
    bits = np.zeros((len(cells), nb, w32 * 32), np.uint8)
    for i, c in enumerate(cells):
        bits[i, :, :nbk] = c["mask"]
    words = np.packbits(bits, axis=2, bitorder="little").view(np.int32).reshape(-1)
    blk_base = np.concatenate([[0], np.cumsum([len(c["blk_idx"]) for c in cells])]).astype(np.int64)
    ivl_base = np.concatenate([[0], np.cumsum([len(c["ivl"]) for c in cells])]).astype(np.int64)
    u16 = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.uint16).view(np.int16)).view(torch.uint16)
    return csa.Plan(lay, len(cells),
                    kind=torch.tensor([c["kind"] for c in cells], dtype=torch.uint8),
                    anchor_k=torch.zeros(len(cells), dtype=torch.int32),
                    mask_bits=torch.from_numpy(words.copy()),
                    blk_base=torch.from_numpy(blk_base),
                    blk_row_ptr=torch.from_numpy(np.concatenate([c["blk_row_ptr"] for c in cells])),
                    blk_idx=u16(np.concatenate([c["blk_idx"] for c in cells])),
                    ivl_base=torch.from_numpy(ivl_base),
                    ivl_row_ptr=torch.from_numpy(np.concatenate([c["ivl_row_ptr"] for c in cells])),
                    ivl=u16(np.concatenate([c["ivl"].reshape(-1) for c in cells])),
                    kept_area=torch.tensor([c["kept_area"] for c in cells], dtype=torch.int64))


@pytest.mark.parametrize("lay", [Layout(2, 5, 25, 64), Layout(2, 9, 40, 128, 80)])
def test_plan_file_round_trip_and_corruption(tmp_path, lay):
    counts = inputs.random_counts(lay.NB, 3, 8, seed=1, nbk=lay.NBK)
    plan = _host_plan(lay, counts, 4)
    path = os.path.join(tmp_path, "plan.csap")
    planio.save_plan(plan, path)
    back = planio.load_plan(path, device="cpu", validate=False)
    assert back.lay == lay and back.n_cells == plan.n_cells
    for name, _ in planio._PLAN_FIELDS:
        a, b = getattr(plan, name), getattr(back, name)
        if a.dtype == torch.uint16:
            a, b = a.view(torch.int16), b.view(torch.int16)
        assert torch.equal(a, b), name
    blob = open(path, "rb").read()
    for bad in (blob[:-9], blob[:20] + bytes([blob[20] ^ 1]) + blob[21:], b"XXXX" + blob[4:]):
        with open(path, "wb") as fh:
            fh.write(bad)
        with pytest.raises(ValueError):
            planio.load_plan(path, device="cpu", validate=False)


def test_intervals_only_plan_file_round_trip(tmp_path):
    """An intervals-only plan (no CSR index) is saved and loaded with an empty
    blk_idx, and its struct hands the kernels a NULL index with capacity 0."""
    lay = Layout(2, 9, 40, 128)
    plan = _host_plan(lay, inputs.random_counts(lay.NB, 2, 8, seed=4), 3)
    plan.blk_idx = torch.empty(0, dtype=torch.int16).view(torch.uint16)
    path = os.path.join(tmp_path, "plan_ivl.csap")
    planio.save_plan(plan, path)
    back = planio.load_plan(path, device="cpu", validate=False)
    assert back.blk_idx.numel() == 0
    assert torch.equal(back.ivl.view(torch.int16), plan.ivl.view(torch.int16))
    st = back.struct()
    assert st.blk_idx is None and st.blk_capacity == 0 and st.ivl_capacity == plan.ivl.numel() // 2


def test_calibration_state_round_trip(tmp_path):
    lay = Layout(2, 9, 40, 128, 96)
    keep = torch.from_numpy(inputs.random_counts(lay.NB, 4, 8, seed=3, nbk=lay.NBK)
                            .reshape(-1).view(np.int16)).view(torch.uint16)
    sim = torch.linspace(0.1, 3.0, 4, dtype=torch.float64)
    path = os.path.join(tmp_path, "cal.csac")
    st = {"T": 50, "L": 40, "H": 4, "anchor_k": 5, "rho": 0.5, "eps_A": 0.842192, "eps_C": 0.99,
          "eps_k": 16.0}
    planio.save_calibration(path, lay, keep, sim, 7, settings=st)
    assert not os.path.exists(path + ".tmp")   # written atomically (tmp + rename)
    lay2, keep2, sim2, n = planio.load_calibration(path, device="cpu", expect=st)
    assert lay2 == lay and n == 7 and torch.equal(sim2, sim)
    assert torch.equal(keep2.view(torch.int16), keep.view(torch.int16))
    for key, val in (("rho", 0.6), ("eps_A", 0.9), ("T", 4), ("anchor_k", 3)):
        with pytest.raises(ValueError, match=key):   # resuming under other settings is refused
            planio.load_calibration(path, device="cpu", expect={**st, key: val})
    with pytest.raises(ValueError):
        planio.save_calibration(path, Layout(2, 9, 40, 128), keep, sim, 7)  # wrong geometry


@pytest.mark.gpu
def test_plan_file_on_gpu_attention_bitwise(tmp_path):
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    lay = Layout(2, 9, 40, 128)
    heads = 3
    counts = inputs.random_counts(lay.NB, heads, 8, seed=9)
    ct = torch.from_numpy(counts.reshape(-1).view(np.int16)).cuda().view(torch.uint16)
    sim = torch.tensor([0.0, 1.0, 0.0], dtype=torch.float64, device="cuda")
    plan = csa.compile_plan(lay, ct, 4, similarity=sim, anchor_k=2)
    path = os.path.join(tmp_path, "p.csap")
    planio.save_plan(plan, path)
    back = planio.load_plan(path)  # validates on the device
    q, k, v = inputs.qkv(1, lay.N, heads, 128, seed=5, device="cuda")
    o1 = csa.sparse_attn_fwd(q, k, v, plan, csa.build_work_list(plan, 0, heads))
    o2 = csa.sparse_attn_fwd(q, k, v, back, csa.build_work_list(back, 0, heads))
    torch.cuda.synchronize()
    assert torch.equal(o1, o2)
    # calibration resumed from a saved state = accumulated in one go
    keep_a = torch.zeros(heads * lay.NB * lay.NB, dtype=torch.int16, device="cuda").view(torch.uint16)
    keep_b = keep_a.clone()
    sim_dummy = torch.zeros(heads, dtype=torch.float64, device="cuda")
    for p in range(2):
        qp, kp, _ = inputs.structured_qk(lay, heads, 128, 1, p, alpha=1.2, device="cuda")
        csa.calib_accumulate(lay, qp, kp, 0.9, keep_a)
        if p == 0:
            csa.calib_accumulate(lay, qp, kp, 0.9, keep_b)
            cpath = os.path.join(tmp_path, "c.csac")
            planio.save_calibration(cpath, lay, keep_b, sim_dummy, 1)
            _, keep_b, _, done = planio.load_calibration(cpath)
            assert done == 1
        else:
            csa.calib_accumulate(lay, qp, kp, 0.9, keep_b)
    torch.cuda.synchronize()
    assert torch.equal(keep_a.view(torch.int16), keep_b.view(torch.int16))
