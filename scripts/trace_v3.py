"""Debug timeline of CTA 0's first item in the single-CTA attention kernel (csa_debug_trace).
Per tile j: group (j & 1) s_full wait / S ready / P published; MMA QK issue and PV p_full wait.
usage: python scripts/trace_v3.py [config].  GPU only."""
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
work = csa.build_work_list(plan, 0, cfg.heads, order=2)
q, k, v = inputs.qkv(1, lay.N, cfg.heads, cfg.d, seed=11, device="cuda")
out = csa.sparse_attn_fwd(q, k, v, plan, work)
buf = torch.zeros(4 * 1024 * 8, dtype=torch.int64, device="cuda")
csa.lib().csa_debug_trace(ctypes.c_void_p(buf.data_ptr()), 0)
csa.sparse_attn_fwd(q, k, v, plan, work, out=out, dynamic=False)
torch.cuda.synchronize()
csa.lib().csa_debug_trace(None, 0)
t = buf.view(4, 1024, 8).cpu().numpy().astype(np.int64)
n = int((t[2, :, 1] > 0).sum())
t0 = t[t > 0].min()
print(f"tiles in CTA 0's first item: {n}")
g = np.array([t[j & 1, j] for j in range(n)])
m = t[2, :n]
sl = slice(8, n - 8)
print(f"group: s_full wait {np.median(g[sl,1]-g[sl,0]):.0f}  softmax (S ready -> P published) "
      f"{np.median(g[sl,2]-g[sl,1]):.0f}  group period {np.median(g[sl,1][2:]-g[sl,1][:-2]):.0f}")
print(f"MMA: kv_full wait {np.median(m[sl,1]-m[sl,0]):.0f}  p_full wait {np.median(m[sl,3]-m[sl,2]):.0f}"
      f"  QK issue period {np.median(np.diff(m[sl,1])):.0f}")
print(f"QK(j) issue -> S(j) ready: {np.median(g[sl,1]-m[sl,1]):.0f}  P(j) published -> PV(j) issued: "
      f"{np.median(m[sl,3]-g[sl,2]):.0f}")
for j in range(20, 28):
    print(j, "grp", [int(x - t0) for x in g[j, :3]], "mma qk", [int(x - t0) for x in m[j, :2]],
          "pv", [int(x - t0) for x in m[j, 2:4]])
