"""Calibration + compile benchmark (BASELINE configs[4]) on B200.

One calibration prompt over every (t, l) cell of the high-step schedule -- 40 layers x 50
timesteps of Wan2.1 14B 480p geometry (21 x 30 x 52 = 32760 tokens, d 128) -- for this rank's
heads: per (t, l), csa_calib_accumulate (a2-a5, single exponential pass, eps(t) from Eq.
eq:epsilon_schedule with A(N), C 0.99, k 16, P:518-526 / P:888-894) and csa_spatial_similarity
(f1) from the pass's own row LSE; then one csa_compile_plan (a6) over all T x L x H_rank cells.
Head-sharded without any collective: under torchrun each rank takes H / WORLD_SIZE
heads; --heads-per-rank emulates one rank of a larger job on a single GPU (5 = one of 8 ranks).

Inputs: generator-G Q/K per (t, l) (head seed 1000 t + l + 1, prompt seed 0, peak-logit scales
spread over the heads, 4 repetitive heads); their generation is timed apart from the calibration
(CUDA events around the library calls only).
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

from paper_2603_05503_b200 import csa, inputs, pipeline  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="wan480")
    ap.add_argument("--layers", type=int, default=40)
    ap.add_argument("--steps-T", type=int, default=50)
    ap.add_argument("--heads-per-rank", type=int, default=0, help="0: H / WORLD_SIZE")
    ap.add_argument("--no-sim", action="store_true")
    ap.add_argument("--separate", action="store_true",
                    help="csa_calib_accumulate + csa_spatial_similarity instead of the fused pass")
    ap.add_argument("--json-out", default=None)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    cfg = inputs.CONFIGS[args.config]
    lay, H, d, L, T = cfg.layout, cfg.heads, cfg.d, args.layers, args.steps_T
    hr = args.heads_per_rank or H // world
    heads = list(range(rank * hr, (rank + 1) * hr))
    alphas = np.linspace(0.8, 1.6, H)[heads]
    rep_all = set(np.linspace(0, H - 1, 4).astype(int).tolist())
    rep = tuple(i for i, h in enumerate(heads) if h in rep_all)
    eps = pipeline.epsilon_schedule(T, *pipeline.high_step_constants(lay.N))
    nb = lay.NB
    cells = T * L * hr
    keep = torch.zeros(cells * nb * nb, dtype=torch.int16, device="cuda").view(torch.uint16)
    sim_sum = torch.zeros(cells, dtype=torch.float64, device="cuda")
    lse = torch.empty(hr * lay.N, dtype=torch.float32, device="cuda")
    ev = []
    gen_s = 0.0
    for t in range(T):
        for l in range(L):
            t0 = time.perf_counter()
            q, k, _ = inputs.structured_qk(lay, hr, d, head_seed=1000 * t + l + 1, prompt_seed=0,
                                           alpha=alphas, repetitive=rep, device="cuda")
            torch.cuda.synchronize()
            gen_s += time.perf_counter() - t0
            c0 = (t * L + l) * hr
            e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            e[0].record()
            if args.no_sim or args.separate:
                csa.calib_accumulate(lay, q, k, eps[t], keep[c0 * nb * nb:(c0 + hr) * nb * nb],
                                     lse_out=lse)
                e[1].record()
                if not args.no_sim:
                    csa.spatial_similarity(lay, q, k, lse, 5, sim_sum[c0:c0 + hr])
            else:  # a2-a5 + f1 in one pass (csa_calib_accumulate_sim); counted as calibration
                csa.calib_accumulate_sim(lay, q, k, eps[t], keep[c0 * nb * nb:(c0 + hr) * nb * nb],
                                         5, sim_sum[c0:c0 + hr])
                e[1].record()
            e[2].record()
            ev.append(e)
            del q, k
    torch.cuda.synchronize()
    calib_ms = sum(e[0].elapsed_time(e[1]) for e in ev)
    sim_ms = sum(e[1].elapsed_time(e[2]) for e in ev)
    s = sim_sum / float(lay.F * lay.H)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = csa.compile_plan(lay, keep, 1, similarity=None if args.no_sim else s, gamma=0.87,
                            anchor_k=5)  # |D| = 1 prompt: rho 0.5 -> min_count 1
    torch.cuda.synchronize()
    compile_ms = (time.perf_counter() - t0) * 1e3
    area = plan.kept_area.double()
    scores = float(T * L * hr) * float(lay.N) ** 2
    sm_mhz = None
    try:
        import subprocess
        sm_mhz = float(subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                                      capture_output=True, text=True).stdout.split()[0])
    except Exception:
        pass
    mufu = 16.0 * torch.cuda.get_device_properties(0).multi_processor_count * (sm_mhz or 1965.0) * 1e6
    out = {
        "workload": f"{cfg.name} geometry, {L} layers x {T} timesteps x {hr} heads (rank {rank} of "
                    f"{world}; {H} heads per layer), d {d}, 1 generator-G prompt, high-step eps(t)",
        "cells": cells, "calib_s_per_prompt": round(calib_ms / 1e3, 3),
        "similarity_s_per_prompt": round(sim_ms / 1e3, 3),
        "calib_qk_tflops": round(2.0 * d * scores / (calib_ms * 1e-3) / 1e12, 1),
        "fused_a2_a5_f1": not (args.no_sim or args.separate),
        # exponentials per score: 1 in csa_calib_accumulate, 2 in the fused pass (p and p_a)
        "calib_exp_per_s": scores * (1 if args.no_sim or args.separate else 2) / (calib_ms * 1e-3),
        "calib_exp_frac_of_mufu": round(scores * (1 if args.no_sim or args.separate else 2)
                                        / (calib_ms * 1e-3) / mufu, 4),
        "mufu_peak_exp_per_s_at_idle_clock": mufu,
        "compile_ms_incl_size_readback": round(compile_ms, 1),
        "keep_count_bytes": keep.numel() * 2, "plan_bytes": plan.nbytes(),
        "mean_kept_fraction": round(float(area.sum().item()) / (cells * float(lay.N) ** 2), 4),
        "repetitive_cells": int(plan.kind.sum().item()),
        "input_generation_s": round(gen_s, 1),
        "eps_range": [round(eps[0], 6), round(eps[-1], 6)],
    }
    print(json.dumps(out), flush=True)
    if args.json_out:
        with open(args.json_out, "w") as fh:
            json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
