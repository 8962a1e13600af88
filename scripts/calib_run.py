"""Run the calibration pass (a2-a5) of one prompt on a bench config; for ncu captures / timing.
usage: python scripts/calib_run.py [config] [iters] [mode: single|two|lse_in]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_05503_b200 import csa, inputs

cfg = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "wan720"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mode = sys.argv[3] if len(sys.argv) > 3 else "single"
lay, H, d = cfg.layout, cfg.heads, cfg.d
q, k, _ = inputs.qkv(1, lay.N, H, d, seed=1, device="cuda")
counts = torch.zeros(H * lay.NB * lay.NB, dtype=torch.int16, device="cuda").view(torch.uint16)
lse = torch.zeros(H * lay.N, dtype=torch.float32, device="cuda") if mode == "lse_in" else None
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for i in range(iters):
    ev[0].record()
    csa.calib_accumulate(lay, q, k, 0.9, counts, lse_in=lse, single_pass=(mode == "single"))
    ev[1].record()
    torch.cuda.synchronize()
    print(f"iter {i}: {ev[0].elapsed_time(ev[1]):.3f} ms")
