"""Debug timeline of the CTA-pair kernel (leader CTA 0): MMA waits and softmax stages."""
import ctypes, os, sys
import numpy as np, torch
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
csa.lib().csa_debug_trace(ctypes.c_void_p(buf.data_ptr()), int(os.environ.get("CSA_DEBUG_MODE", "0")))
csa.sparse_attn_fwd(q, k, v, plan, work, out=out)
torch.cuda.synchronize()
csa.lib().csa_debug_trace(None, 0)
t = buf.view(4, 1024, 8).cpu().numpy().astype(np.int64)
np.save("gpurun_out/trace_pair.npy", t)
t0 = t[t > 0].min()
S, P = t[2], t[3]
ok = (S[:, 3] > 0) & (P[:, 3] > 0)
idx = np.nonzero(ok)[0][20:300]
print("S: s_free wait", np.median(S[idx, 1] - S[idx, 0]), " kv wait", np.median(S[idx, 2] - S[idx, 1]),
      " issue", np.median(S[idx, 3] - S[idx, 2]))
print("PV: p_full wait", np.median(P[idx, 1] - P[idx, 0]), " kv wait", np.median(P[idx, 2] - P[idx, 1]),
      " issue", np.median(P[idx, 3] - P[idx, 2]))
print("S period", np.median(np.diff(S[idx, 0])), " PV period", np.median(np.diff(P[idx, 0])))
for g in (0, 1):
    a = t[g][(t[g][:, 4] > 0)][20:300]
    print(f"half {g}: busy {np.median(a[:, 4] - a[:, 0]):.0f} period {np.median(np.diff(a[:, 0])):.0f}")
for j in range(100, 106):
    print(j, "S", [int(x - t0) for x in S[j, :4]], "PV", [int(x - t0) for x in P[j, :4]],
          "sm0", [int(x - t0) for x in t[0, j, [0, 4]]])
