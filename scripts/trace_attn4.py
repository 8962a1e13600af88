"""Debug timeline of CTA 0's first 1024 tiles in the fixed-reference attention kernel (attn4.cu;
trace build: CSA_TRACE_BUILD=1).  Per tile: softmax group g: s_full wait start / S ready / S
loaded / P computed+stored / P published; QK issue: K wait start / K ready; PV issue: p_full
wait start / P ready / issued.  usage: trace_attn4.py [config]  (CSA_DEBUG_MODE=1: no exp)"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_05503_b200 import csa, inputs  # noqa: E402

os.environ["CSA_ATTN4"] = "1"  # attn5.cu is the default path

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
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
csa.sparse_attn_fwd(q, k, v, plan, work, out=out)
e1.record()
torch.cuda.synchronize()
csa.lib().csa_debug_trace(None, 0)
print(f"launch {e0.elapsed_time(e1):.3f} ms")
t = buf.view(4, 1024, 8).cpu().numpy().astype(np.int64)
g0, g1, qk, pv = t[0], t[1], t[2], t[3]
n = int((qk[:, 1] > 0).sum())
sl = slice(16, n - 16)
print(f"tiles {n}; per-tile period (QK issue) {np.median(np.diff(qk[sl, 1])):.0f} cycles")
for nm, g, par in (("group0", g0, 0), ("group1", g1, 1)):
    rows = np.array([i for i in range(16, n - 16) if g[i, 1] > 0])
    d = lambda a, b: np.median(g[rows, b] - g[rows, a])
    per = np.median(np.diff(g[rows, 1]))
    print(f"{nm} ({len(rows)} tiles, period {per:.0f}): s_full wait {d(0,1):.0f}  ld {d(1,2):.0f}  "
          f"compute+st {d(2,3):.0f}  st_wait+publish {d(3,4):.0f}")
    # gap from this tile's publish to the group's next S ready
    nxt = np.median([g[rows[i + 1], 1] - g[rows[i], 4] for i in range(len(rows) - 1)])
    print(f"   P published -> next S ready {nxt:.0f}")
print(f"QK issuer: K wait {np.median(qk[sl,1]-qk[sl,0]):.0f}")
print(f"PV issuer: p_full wait {np.median(pv[sl,1]-pv[sl,0]):.0f}  V wait+issue {np.median(pv[sl,2]-pv[sl,1]):.0f}")
t0 = t[t > 0].min()
for j in range(40, 48):
    g = g0 if g0[j, 1] > 0 else g1
    print(j, "grp", 0 if g0[j, 1] > 0 else 1, [int(x - t0) for x in g[j, :5]], "QK", [int(x - t0) for x in qk[j, :2]],
          "PV", [int(x - t0) for x in pv[j, :3]])
