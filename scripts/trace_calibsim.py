"""Debug timeline of CTA 0 in calibsim.cu (trace build): per row group, S wait start / S ready /
last chunk loaded (S released) / tile done; MMA issuer: s_empty wait start / S free / K ready /
issued."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_05503_b200 import csa, inputs  # noqa: E402

cfg = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "wan720"]
lay = cfg.layout
H = cfg.heads
q, k, _ = inputs.qkv(1, lay.N, H, cfg.d, seed=11, device="cuda")
cnt = torch.zeros(H * lay.NB * lay.NBK, dtype=torch.int16, device="cuda").view(torch.uint16)
sim = torch.zeros(H, dtype=torch.float64, device="cuda")
csa.calib_accumulate_sim(lay, q, k, 0.9, cnt, 5, sim)
buf = torch.zeros(4 * 1024 * 8, dtype=torch.int64, device="cuda")
csa.lib().csa_debug_trace(ctypes.c_void_p(buf.data_ptr()), 0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
csa.calib_accumulate_sim(lay, q, k, 0.9, cnt, 5, sim)
e1.record()
torch.cuda.synchronize()
csa.lib().csa_debug_trace(None, 0)
print(f"launch {e0.elapsed_time(e1):.3f} ms")
t = buf.view(4, 1024, 8).cpu().numpy().astype(np.int64)
base = int(t[2][0, 0])
for g in range(2):
    sm = t[g]
    n = int((sm[:, 1] > 0).sum())
    sl = slice(16, min(n, 280) - 16)
    d = lambda a, b: np.median(sm[sl, b] - sm[sl, a])
    print(f"group {g}: tiles {n}; period {np.median(np.diff(sm[sl, 1])):.0f}: S wait {d(0,1):.0f} "
          f"chunks to release {d(1,2):.0f} rest {d(2,3):.0f}; release -> next S ready "
          f"{np.median(sm[17:min(n,280)-15, 1] - sm[16:min(n,280)-16, 2]):.0f}")
mm = t[2]
sl = slice(32, 500)
print(f"MMA: s_empty wait {np.median(mm[sl,1]-mm[sl,0]):.0f} K wait {np.median(mm[sl,2]-mm[sl,1]):.0f} "
      f"issue {np.median(mm[sl,3]-mm[sl,2]):.0f}")
for j in range(40, 46):
    print(j, "MMA", [int(x - base) for x in mm[j, :4]])
for j in range(20, 23):
    print(j, "G0", [int(x - base) for x in t[0][j, :4]], "G1", [int(x - base) for x in t[1][j, :4]])
