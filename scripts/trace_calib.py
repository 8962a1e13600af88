"""Debug timeline of CTA 0's first item in the calibration kernel (csa_debug_trace).
usage: python scripts/trace_calib.py [config] [mode single|two|lse_in].  GPU only."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_05503_b200 import csa, inputs  # noqa: E402

cfg = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "wan720"]
mode = sys.argv[2] if len(sys.argv) > 2 else "single"
lay, H, d = cfg.layout, cfg.heads, cfg.d
q, k, _ = inputs.qkv(1, lay.N, H, d, seed=1, device="cuda")
counts = torch.zeros(H * lay.NB * lay.NB, dtype=torch.int16, device="cuda").view(torch.uint16)
lse = torch.zeros(H * lay.N, dtype=torch.float32, device="cuda") if mode == "lse_in" else None
run = lambda: csa.calib_accumulate(lay, q, k, 0.9, counts, lse_in=lse, single_pass=(mode == "single"))
run()
buf = torch.zeros(4 * 1024 * 8, dtype=torch.int64, device="cuda")
csa.lib().csa_debug_trace(ctypes.c_void_p(buf.data_ptr()), int(os.environ.get("CSA_DEBUG_MODE", "0")))
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record()
run()
ev[1].record()
torch.cuda.synchronize()
print(f"mode {os.environ.get('CSA_DEBUG_MODE', '0')}: kernel {ev[0].elapsed_time(ev[1]):.2f} ms")
csa.lib().csa_debug_trace(None, 0)
t = buf.view(4, 1024, 8).cpu().numpy().astype(np.int64)
t0 = t[t > 0].min()
n = min(lay.NB, 1024)
for g in (0, 1):
    a = t[g][g:n:2]
    a = a[(a[:, 1] > 0)][10:-10]
    print(f"group {g}: tiles {len(a)}  s_full wait {np.median(a[:,1]-a[:,0]):.0f}  ld+release "
          f"{np.median(a[:,2]-a[:,1]):.0f}  compute {np.median(a[:,3]-a[:,2]):.0f}  period "
          f"{np.median(np.diff(a[:,1])):.0f}")
m = t[2][:n]
m = m[m[:, 2] > 0][10:-10]
print(f"MMA: s_empty wait {np.median(m[:,1]-m[:,0]):.0f}  k_full wait {np.median(m[:,2]-m[:,1]):.0f}"
      f"  issue period {np.median(np.diff(m[:,2])):.0f}")
p = t[3][:n]
p = p[p[:, 1] > 0][10:-10]
print(f"TMA: k_empty wait {np.median(p[:,1]-p[:,0]):.0f}  period {np.median(np.diff(p[:,1])):.0f}")
for j in range(40, 48):
    print(j, "grp", [int(x - t0) for x in t[j & 1, j, :4]], "mma", [int(x - t0) for x in t[2, j, :3]],
          "tma", [int(x - t0) for x in t[3, j, :2]])
