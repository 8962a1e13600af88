"""Host-side logic on CPU: the synthetic plan generator (generator S) on square and non-square
grids, the bench's FLOP accounting against the oracle compiler's kept area, and the head
balancing used by the multi-GPU bench."""
import os

import numpy as np
import pytest

import oracle
from paper_2603_05503_b200 import inputs, ulysses
from paper_2603_05503_b200.inputs import Layout


@pytest.mark.parametrize("lay,target", [(Layout(6, 10, 16, 32), 0.6), (Layout(6, 10, 16, 32, 48), 0.5),
                                        (Layout(21, 30, 52, 128), 0.68)])
def test_generator_s_sparsity_diagonal_and_sink(lay, target):
    heads = 4
    m = inputs.synthetic_masks(lay, heads, target, seed=1)
    assert m.shape == (heads, lay.NB, lay.NBK)
    qs = np.array([lay.block_size(r) for r in range(lay.NB)])
    ks = np.array([lay.key_block_size(c) for c in range(lay.NBK)])
    sp = 1.0 - np.einsum("hrc,r,c->", m.astype(np.int64), qs, ks) / (heads * float(lay.N) ** 2)
    assert abs(sp - target) <= 0.005 + 1e-9
    assert (m[:, :, 0] == 1).all()  # sink key block
    centre = (np.arange(lay.NB) * lay.B + (qs - 1) // 2) // lay.Bkv
    assert (m[:, np.arange(lay.NB), centre] == 1).all()  # the query block's own keys


def test_generator_s_masks_are_nested_in_the_sparsity():
    """Same seed, lower target sparsity -> superset (what the compaction bench relies on for its
    timestep drift)."""
    lay = Layout(21, 30, 52, 128)
    a = inputs.synthetic_masks(lay, 4, 0.65, seed=0)
    b = inputs.synthetic_masks(lay, 4, 0.55, seed=0)
    assert (b >= a).all() and (b > a).any()


def test_bench_flop_accounting_equals_oracle_kept_area():
    import bench

    lay = Layout(3, 7, 100, 128)
    masks = inputs.synthetic_masks(lay, 3, 0.6, seed=2)
    rep = {1}
    for h in range(3):
        flop, area = bench.flops_of(lay, masks, rep, [h], 128, 2)
        if h in rep:
            assert area == lay.F * 5 * lay.W * lay.N
        else:
            cell = oracle.compile_cell(masks[h].astype(np.uint16) * 64, lay.N, lay.B, lay.F,
                                       lay.H, lay.W, 32)
            assert area == cell["kept_area"]
        assert flop == 4.0 * 128 * 2 * area


def test_balance_heads_on_bench_costs():
    import bench

    cfg = inputs.CONFIGS["wan480"]
    masks = inputs.synthetic_masks(cfg.layout, cfg.heads, cfg.sparsity, seed=0)
    rep = set(np.linspace(0, cfg.heads - 1, 4).astype(int).tolist())
    cost = [bench.flops_of(cfg.layout, masks, rep, [h], 128, 1)[1] for h in range(cfg.heads)]
    for world in (2, 4, 8):
        perm = ulysses.balance_heads(cost, world)
        hp = cfg.heads // world
        loads = [sum(cost[h] for h in perm[r * hp:(r + 1) * hp]) for r in range(world)]
        nat = [sum(cost[r * hp:(r + 1) * hp]) for r in range(world)]
        assert sorted(perm) == list(range(cfg.heads))
        assert max(loads) <= max(nat) and max(loads) / (sum(cost) / world) < 1.03


def test_bench_multi_gpu_request_fails_loudly_without_gpus():
    """`bench.py --gpus 2` outside torchrun with fewer than 2 visible GPUs must refuse (never
    report a smaller job under a larger n_gpus)."""
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    res = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2",
                          "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                         env=env, timeout=300)
    assert res.returncode != 0
    assert "refusing" in res.stderr + res.stdout
