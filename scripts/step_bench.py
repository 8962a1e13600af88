"""Denoising-step benchmark (f4): the attention of all layers of one step, CFG batch 2, from a
calibrated T x L x H plan dictionary, eager vs CUDA-graph replay, on one B200.

Workload (DESIGN.md f4): Wan2.1 14B 480p geometry (21 x 30 x 52 = 32760 tokens, 40 heads,
d 128, 40 layers), 4-step distilled schedule (A, C, k) = (0.763, 0.863, 5.64), |D|
generator-G prompts (conditional branch only; per-(t, l) head seeds, peak-logit scales
spread over heads, 4 repetitive heads per layer), rho 0.5, gamma 0.87, k 5.  Inference inputs:
seeded N(0,1) bf16 Q/K/V [2, N, 40, 128] in --sets rotating buffer sets (each set 2 GB > L2).
Reported per step t: kept fraction, eager and graph ms for the 40 layers, effective TFLOP/s of
the kept FLOPs, and the same step on the all-ones dictionary (dense) -> speedup.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_05503_b200 import csa, inputs, pipeline  # noqa: E402


def timed(fn, steps, warmup):
    for _ in range(warmup):
        fn()
    ts = []
    for _ in range(steps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="wan480")
    ap.add_argument("--layers", type=int, default=40)
    ap.add_argument("--steps-T", type=int, default=4)
    ap.add_argument("--prompts", type=int, default=2)
    ap.add_argument("--sets", type=int, default=4)
    ap.add_argument("--batch", type=int, default=2)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--json-out", default=None)
    args = ap.parse_args()
    cfg = inputs.CONFIGS[args.config]
    lay, H, d, L, T = cfg.layout, cfg.heads, cfg.d, args.layers, args.steps_T
    rep = tuple(np.linspace(0, H - 1, 4).astype(int).tolist())
    alphas = np.linspace(0.8, 1.6, H)

    def qk(p, t, l):
        q, k, _ = inputs.structured_qk(lay, H, d, head_seed=1000 * t + l + 1, prompt_seed=p,
                                       alpha=alphas, repetitive=rep, device="cuda")
        return q, k

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dic = pipeline.calibrate(lay, T, L, H, args.prompts, qk, pipeline.DISTILLED)
    torch.cuda.synchronize()
    calib_s = time.perf_counter() - t0
    n_rep = int(dic.plan.kind.sum().item())
    bufs = [inputs.qkv(args.batch, lay.N, H, d, seed=200 + s, device="cuda")
            for s in range(args.sets)]
    outs = [torch.empty_like(b[0]) for b in bufs]
    step = pipeline.DenoiseStep(dic, [b[0] for b in bufs], [b[1] for b in bufs],
                                [b[2] for b in bufs], outs)
    # dense comparator: all-ones counts for one step's cells
    nb = lay.NB
    ones = torch.full((L * H * nb * nb,), 64, dtype=torch.int16, device="cuda").view(torch.uint16)
    plan1 = csa.compile_plan(lay, ones, 32)
    dense_dic = pipeline.PlanDictionary(lay, 1, L, H, plan1, [1.0], 32, 1,
                                        torch.zeros(L * H, dtype=torch.float64, device="cuda"),
                                        ones.view(L * H, nb, nb))
    dense = pipeline.DenoiseStep(dense_dic, [b[0] for b in bufs], [b[1] for b in bufs],
                                 [b[2] for b in bufs], outs)
    ms_dense = timed(lambda: dense.replay(0), max(2, args.iters // 2), 1)
    rows = []
    for t in range(T):
        ms_eager = timed(lambda: step.run(t), args.iters, 2)
        ms_graph = timed(lambda: step.replay(t), args.iters, 2)
        flop = step.flop(t)
        row = {"t": t, "eps": round(dic.eps[t], 6), "kept_fraction": round(dic.kept_fraction(t), 4),
               "layers": L, "batch": args.batch, "eager_ms": round(ms_eager, 3),
               "graph_ms": round(ms_graph, 3),
               "tflops_eff_graph": round(flop / (ms_graph * 1e-3) / 1e12, 1),
               "dense_graph_ms": round(ms_dense, 3),
               "speedup_vs_dense": round(ms_dense / ms_graph, 3),
               "kernels_per_step": 2 * L}
        rows.append(row)
        print(json.dumps(row), flush=True)
    total = sum(r["graph_ms"] for r in rows)
    summary = {"workload": f"{cfg.name} geometry, {L} layers x {H} heads, d {d}, {T}-step distilled "
                           f"schedule (P:886), CFG batch {args.batch}, |D| = {args.prompts}",
               "calibration_s": round(calib_s, 2), "cells": T * L * H, "repetitive_cells": n_rep,
               "plan_bytes": dic.plan.nbytes(), "mean_kept_fraction": round(dic.kept_fraction(), 4),
               "attention_ms_all_steps_graph": round(total, 2),
               "dense_ms_all_steps": round(T * ms_dense, 2),
               "speedup_all_steps": round(T * ms_dense / total, 3), "steps": rows}
    print(json.dumps({k: v for k, v in summary.items() if k != "steps"}), flush=True)
    if args.json_out:
        with open(args.json_out, "w") as fh:
            json.dump(summary, fh, indent=1)


if __name__ == "__main__":
    main()
