"""Debug timeline of CTA 0 in attn6.cu (trace build; pair items): per group, softmax (S wait
start / S ready / S loaded / exps + P stores issued / P published) and MMA issuer (p_full wait
start / P ready / V ready / P.V issued / next S-MMA issued)."""
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
work = csa.build_work_list(plan, 0, cfg.heads, order=3)
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
base = min(int(t[s][0, 0]) for s in range(4) if t[s][0, 0] > 0)
for g in range(2):
    sm, mm = t[g], t[2 + g]
    n = int((sm[:, 1] > 0).sum())
    sl = slice(16, n - 16)
    d = lambda a, b: np.median(sm[sl, b] - sm[sl, a])
    print(f"group {g}: tiles {n}; softmax period {np.median(np.diff(sm[sl, 1])):.0f}: S wait {d(0,1):.0f} "
          f"ld {d(1,2):.0f} exp+st {d(2,3):.0f} st_wait+publish {d(3,4):.0f}")
    dm = lambda a, b: np.median(mm[sl, b] - mm[sl, a])
    print(f"  MMA: p wait {dm(0,1):.0f} V wait {dm(1,2):.0f} PV issue {dm(2,3):.0f} QK wait+issue {dm(3,4):.0f}; "
          f"P published -> next S ready {np.median(sm[17:n-15, 1] - sm[16:n-16, 4]):.0f}")
    for j in range(40, 44):
        print(" ", j, "SM", [int(x - base) for x in sm[j, :5]], "MMA", [int(x - base) for x in mm[j, :5]])
