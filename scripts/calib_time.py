"""Time the calibration passes per config (python calib_time.py [configs]): a2-a5 single
exponential pass, f1 similarity pass, and the fused a2-a5 + f1 pass (csa_calib_accumulate_sim)."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_05503_b200 import csa, inputs  # noqa: E402


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


for name in sys.argv[1:] or ["wan720", "wan480"]:
    cfg = inputs.CONFIGS[name]
    lay = cfg.layout
    H = cfg.heads
    q, k, _ = inputs.qkv(1, lay.N, H, cfg.d, seed=11, device="cuda")
    cnt = torch.zeros(H * lay.NB * lay.NBK, dtype=torch.int16, device="cuda").view(torch.uint16)
    lse = torch.empty(H * lay.N, dtype=torch.float32, device="cuda")
    sim = torch.zeros(H, dtype=torch.float64, device="cuda")
    eps = 0.9
    t_cal = timed(lambda: csa.calib_accumulate(lay, q, k, eps, cnt, lse_out=lse))
    t_sim = timed(lambda: csa.spatial_similarity(lay, q, k, lse, 5, sim))
    t_fused = timed(lambda: csa.calib_accumulate_sim(lay, q, k, eps, cnt, 5, sim))
    exps = H * float(lay.N) ** 2
    print(f"{name}: calib {t_cal:.2f} ms ({exps / t_cal / 1e9:.3f} Texp/s), similarity "
          f"{t_sim:.2f} ms, two calls {t_cal + t_sim:.2f} ms; fused {t_fused:.2f} ms "
          f"({2 * exps / t_fused / 1e9:.3f} Texp/s)")
