"""Debug timeline of CTA 0's first 1024 tiles in attn5.cu (trace build): softmax
(S wait start / S ready / S loaded / exps done / P published), QK issue (s_empty wait start /
K ready), PV issue (p_full wait start / P ready / issued)."""
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
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
csa.sparse_attn_fwd(q, k, v, plan, work, out=out)
e1.record()
torch.cuda.synchronize()
csa.lib().csa_debug_trace(None, 0)
print(f"launch {e0.elapsed_time(e1):.3f} ms")
t = buf.view(4, 1024, 8).cpu().numpy().astype(np.int64)
sm, qk, pv = t[0], t[2], t[3]
n = int((sm[:, 1] > 0).sum())
sl = slice(16, n - 16)
d = lambda a, b: np.median(sm[sl, b] - sm[sl, a])
print(f"tiles {n}; softmax period {np.median(np.diff(sm[sl, 1])):.0f}: S wait {d(0,1):.0f} "
      f"ld {d(1,2):.0f} exp {d(2,3):.0f} P store+publish {d(3,4):.0f}; "
      f"published -> next S ready {np.median(sm[17:n-15, 1] - sm[16:n-16, 4]):.0f}")
print(f"QK: s_empty+K wait {np.median(qk[sl,1]-qk[sl,0]):.0f}; PV: p_full wait "
      f"{np.median(pv[sl,1]-pv[sl,0]):.0f}, issue {np.median(pv[sl,2]-pv[sl,1]):.0f}")
t0 = sm[40, 0]
for j in range(40, 46):
    print(j, "SM", [int(x - t0) for x in sm[j, :5]], "QK", [int(x - t0) for x in qk[j, :2]],
          "PV", [int(x - t0) for x in pv[j, :3]])
