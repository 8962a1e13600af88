"""Time one calibration pass (a2-a5, single exponential pass) per config: python calib_time.py."""
import math
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_05503_b200 import csa, inputs  # noqa: E402

for name in sys.argv[1:] or ["wan720", "wan480"]:
    cfg = inputs.CONFIGS[name]
    lay = cfg.layout
    q, k, _ = inputs.qkv(1, lay.N, cfg.heads, cfg.d, seed=11, device="cuda")
    cnt = torch.zeros(cfg.heads * lay.NB * lay.NBK, dtype=torch.int16, device="cuda").view(torch.uint16)
    eps = 0.9
    for _ in range(2):
        csa.calib_accumulate(lay, q, k, eps, cnt)
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        csa.calib_accumulate(lay, q, k, eps, cnt)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = statistics.median(ts)
    exps = cfg.heads * float(lay.N) ** 2
    print(f"{name}: {ms:.2f} ms, {exps / ms / 1e9:.3f} Texp/s")
