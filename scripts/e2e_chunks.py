import sys, time, statistics
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2603_05503_b200 import csa, inputs
cfg = inputs.CONFIGS['wan720']; lay = cfg.layout
masks = inputs.synthetic_masks(lay, cfg.heads, cfg.sparsity, seed=0)
cnt = torch.from_numpy((masks.astype(np.uint16) * np.uint16(64)).reshape(-1).view(np.int16)).cuda().view(torch.uint16)
plan = csa.compile_plan(lay, cnt, 32)
q, k, v = inputs.qkv(1, lay.N, cfg.heads, cfg.d, seed=11, device='cuda')
hq, hk, hv = (t.cpu().pin_memory() for t in (q, k, v))
ho = torch.empty(q.shape, dtype=q.dtype).pin_memory()
for hpc in (2, 1):
    for _ in range(2):
        csa.sparse_attn_fwd_host(hq, hk, hv, plan, ho, heads_per_chunk=hpc)
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); csa.sparse_attn_fwd_host(hq, hk, hv, plan, ho, heads_per_chunk=hpc); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(hpc, round(statistics.median(ts), 2), 'ms')
