"""Attention launch time with the softmax arithmetic on (mode 0) and off (mode 1): the gap shows
how much of the step the MMA/TMA pipeline alone costs.  GPU only, debug."""
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
plan = csa.compile_plan(lay, cnt.view(torch.uint16), 32, csr=os.environ.get("CSR", "1") == "1")
work = csa.build_work_list(plan, 0, cfg.heads, order=int(os.environ.get("ORDER", "3")))
D = int(os.environ.get("D", cfg.d))
q, k, v = inputs.qkv(1, lay.N, cfg.heads, D, seed=11, device="cuda")
out = torch.empty_like(q)
sizes = np.array([lay.block_size(c) for c in range(lay.NB)], np.int64)
flop = 4.0 * D * float(np.einsum("hrc,r,c->", masks.astype(np.int64), sizes, sizes))
modes = [int(x) for x in os.environ.get("MODES", "0,1,2,3,4").split(",")]
for mode in modes:
    csa.lib().csa_debug_trace(None, mode)
    for _ in range(3):
        csa.sparse_attn_fwd(q, k, v, plan, work, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        csa.sparse_attn_fwd(q, k, v, plan, work, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"mode {mode}: {ms:.3f} ms  {flop / ms / 1e9:.1f} TFLOP/s")
csa.lib().csa_debug_trace(None, 0)
