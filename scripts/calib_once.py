"""One launch each of the calibration kernels on a config (for ncu captures):
csa_calib_accumulate (single pass, calib_kernel) then csa_calib_accumulate_sim (calib_sim_kernel)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_05503_b200 import csa, inputs  # noqa: E402

cfg = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "wan720"]
lay = cfg.layout
H = cfg.heads
q, k, _ = inputs.qkv(1, lay.N, H, cfg.d, seed=11, device="cuda")
cnt = torch.zeros(H * lay.NB * lay.NBK, dtype=torch.int16, device="cuda").view(torch.uint16)
sim = torch.zeros(H, dtype=torch.float64, device="cuda")
csa.calib_accumulate(lay, q, k, 0.9, cnt)
csa.calib_accumulate_sim(lay, q, k, 0.9, cnt, 5, sim)
torch.cuda.synchronize()
print("ok")
