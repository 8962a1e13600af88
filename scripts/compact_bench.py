"""Plan-compaction benchmark (f2, Table tab:skip_list_memory).

One Wan2.1 720p layer's plan dictionary over T = 50 timesteps x 40 heads (2000 cells, N_B = 591):
per head, generator-S masks whose sparsity follows the timestep (0.55 at t = 0 rising to 0.65,
shape of Eq. eq:epsilon_schedule with k = 16: later steps sparser and nearly identical); the
masks are nested across t (same seed, growing distance cut), as calibrated masks drift. Counts
= 64 M, rho 0.5.  Measured on the GPU kernels (csa_merge_intervals, csa_share_timesteps,
csa_compile_plan):
  * the 1D skip-list footprint of the layer = sum over STORED masks of 4 B per interval
    (uint16 start/end) + 4 B per row pointer; with timestep sharing a clique's mask is stored
    once; extrapolated x 40 layers for the whole dictionary (the paper's GB column);
  * kept fraction (area) after merging / sharing, blocks added, kernel times.
Rows: merge percentile 100 (none), 99, 95, 90, and 90 with tau 0.98 / 0.97 (the paper's rows).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_05503_b200 import csa, inputs  # noqa: E402


def measure(lay, counts, H, T, clusters=None):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = csa.compile_plan(lay, counts, 32)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    nb = lay.NB
    irp = plan.ivl_row_ptr.view(T * H, nb + 1)[:, -1].cpu().numpy().astype(np.int64)
    per_mask = 4 * irp + 4 * (nb + 1)
    if clusters is None:
        stored = per_mask.sum()
        n_masks = T * H
    else:
        cl = clusters.cpu().numpy()  # [H, T]
        stored, n_masks = 0, 0
        for h in range(H):
            seen = set()
            for t in range(T):
                if cl[h, t] not in seen:
                    seen.add(cl[h, t])
                    stored += per_mask[t * H + h]
                    n_masks += 1
    area = plan.kept_area.double().sum().item()
    return plan, {"intervals": int(irp.sum()), "stored_masks": int(n_masks),
                  "layer_bytes_1d": int(stored),
                  "dictionary_gb_1d_x40_layers": round(40 * stored / 1e9, 3),
                  "kept_fraction": round(area / (T * H * float(lay.N) ** 2), 5),
                  "compile_ms": round(ms, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps-T", type=int, default=50)
    ap.add_argument("--json-out", default=None)
    args = ap.parse_args()
    cfg = inputs.CONFIGS["wan720"]
    lay, H, T = cfg.layout, cfg.heads, args.steps_T
    nb = lay.NB
    sp = [0.55 + 0.10 * (1.0 - math.exp(-16.0 * t / T)) for t in range(T)]
    host = np.empty((T, H, nb, nb), np.uint16)
    cache = {}
    for t in range(T):
        key = round(sp[t], 4)
        if key not in cache:
            cache[key] = inputs.synthetic_masks(lay, H, key, seed=0).astype(np.uint16) * np.uint16(64)
        host[t] = cache[key]
    counts0 = torch.from_numpy(host.reshape(-1).view(np.int16)).cuda().view(torch.uint16)
    del host
    rows = []
    plan0, base = measure(lay, counts0, H, T)
    rows.append({"merge_pct": 100, "tau": None, **base})
    merged = {}
    for pct in (99, 95, 90):
        c = counts0.clone()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        target, added = csa.merge_intervals(plan0, c, 32, float(pct))
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        plan, m = measure(lay, c, H, T)
        merged[pct] = (plan, c)
        rows.append({"merge_pct": pct, "tau": None, "target_width": int(target.item()),
                     "blocks_added": int(added.item()), "merge_ms": round(ms, 2), **m})
    plan90, c90 = merged[90]
    for tau in (0.98, 0.97):
        c = c90.clone()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cluster, _ = csa.share_timesteps(plan90, c, H, T, 32, tau)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        _, m = measure(lay, c, H, T, clusters=cluster)
        rows.append({"merge_pct": 90, "tau": tau, "share_ms": round(ms, 2), **m})
    b0 = rows[0]["layer_bytes_1d"]
    for r in rows:
        r["reduction_vs_no_merge"] = round(1.0 - r["layer_bytes_1d"] / b0, 4)
        print(json.dumps(r), flush=True)
    if args.json_out:
        with open(args.json_out, "w") as fh:
            json.dump({"workload": f"wan720 one layer, {H} heads x {T} timesteps (generator-S "
                                   "masks, sparsity 0.55 -> 0.65 over t, nested), rho 0.5",
                       "rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
