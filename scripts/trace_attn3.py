"""Debug timeline of CTA 0's first item in the Q-in-TMEM attention kernel (attn3.cu).
Per tile j: softmax half h: s_full wait start / S ready / P published; S-issuer: s_free wait
start / K ready (issue); PV-issuer: p_full wait start / P ready.  usage: trace_attn3.py [config]"""
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
csa.lib().csa_debug_trace(ctypes.c_void_p(buf.data_ptr()), int(os.environ.get("CSA_DEBUG_MODE", "0")))
csa.sparse_attn_fwd(q, k, v, plan, work, out=out, dynamic=False)
torch.cuda.synchronize()
csa.lib().csa_debug_trace(None, 0)
t = buf.view(4, 1024, 8).cpu().numpy().astype(np.int64)
n = int((t[2, :, 1] > 0).sum())
t0 = t[t > 0].min()
sl = slice(8, n - 8)
h0, h1, si, pv = t[0, :n], t[1, :n], t[2, :n], t[3, :n]
print(f"tiles {n}; per-tile period (S issue) {np.median(np.diff(si[sl,1])):.0f} cycles")
for nm, h in (("half0", h0), ("half1", h1)):
    print(f"{nm}: s_full wait {np.median(h[sl,1]-h[sl,0]):.0f}  S ready -> P published "
          f"{np.median(h[sl,2]-h[sl,1]):.0f}")
print(f"S-issuer: wait (s_free + k_full) {np.median(si[sl,1]-si[sl,0]):.0f}; issue -> S ready "
      f"{np.median(h0[sl,1]-si[sl,1]):.0f}")
print(f"PV-issuer: p_full wait {np.median(pv[sl,1]-pv[sl,0]):.0f}")
for j in range(20, 26):
    print(j, "h0", [int(x - t0) for x in h0[j, :3]], "h1", [int(x - t0) for x in h1[j, :3]],
          "S", [int(x - t0) for x in si[j, :2]], "PV", [int(x - t0) for x in pv[j, :2]])
for nm, h in (("half0", h0), ("half1", h1)):
    d = lambda a, b: np.median(h[sl, b] - h[sl, a])
    print(f"{nm}: ld {d(1,3):.0f}  exp {d(3,4):.0f}  max+barrier {d(4,5):.0f}  "
          f"p_empty {d(5,6):.0f}  store+publish {d(6,2):.0f}")
