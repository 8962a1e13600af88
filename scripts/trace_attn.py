"""Debug timeline of CTA 0 of the attention kernel (csa_debug_trace) at a BASELINE config.

Prints per-tile durations of the softmax stages and the MMA waits.  GPU only."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_05503_b200 import csa, inputs  # noqa: E402

cfg = inputs.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "wan720"]
lay = cfg.layout
masks = inputs.synthetic_masks(lay, cfg.heads, cfg.sparsity or 0.69, seed=0)
cnt = torch.from_numpy((masks.astype(np.uint16) * np.uint16(64)).reshape(-1).view(np.int16)).cuda()
plan = csa.compile_plan(lay, cnt.view(torch.uint16), 32)
work = csa.build_work_list(plan, 0, cfg.heads)
q, k, v = inputs.qkv(1, lay.N, cfg.heads, cfg.d, seed=11, device="cuda")
out = csa.sparse_attn_fwd(q, k, v, plan, work)
buf = torch.zeros(4 * 1024 * 8, dtype=torch.int64, device="cuda")
csa.lib().csa_debug_trace(ctypes.c_void_p(buf.data_ptr()), int(os.environ.get("CSA_DEBUG_MODE", "0")))
csa.sparse_attn_fwd(q, k, v, plan, work, out=out)
torch.cuda.synchronize()
csa.lib().csa_debug_trace(None, 0)
t = buf.view(4, 1024, 8).cpu().numpy().astype(np.int64)
os.makedirs("gpurun_out", exist_ok=True)
np.save("gpurun_out/trace.npy", t)
t0 = t[t > 0].min()
for g in (0, 1):
    a = t[g]
    ok = (a[:, 4] > 0)
    a = a[ok][20:400]
    print(f"half {g}: tiles {ok.sum()}  ld {np.median(a[:,1]-a[:,0]):.0f}  exp+max+bar {np.median(a[:,2]-a[:,1]):.0f}"
          f"  pwait+st {np.median(a[:,3]-a[:,2]):.0f}  arrive {np.median(a[:,4]-a[:,3]):.0f}"
          f"  busy {np.median(a[:,4]-a[:,0]):.0f}  period {np.median(np.diff(a[:,0])):.0f}")
s = t[2][t[2][:, 0] > 0][20:400, 0]
pv = t[3][t[3][:, 1] > 0][20:400]
print(f"S issue period {np.median(np.diff(s)):.0f}; PV p_full wait {np.median(pv[:,1]-pv[:,0]):.0f}"
      f"  PV period {np.median(np.diff(pv[:,1])):.0f}")
for j in range(80, 88):
    print(j, [int(x - t0) for x in t[0, j, :5]], [int(x - t0) for x in t[1, j, :5]],
          "S", int(t[2, j, 0] - t0), "PVp", int(t[3, j, 0] - t0), int(t[3, j, 1] - t0))
