"""Quick GPU check of the CTA-pair attention kernel against the oracle and the single-CTA kernel.
Run under `timeout`.  Prints max/mean errors; exits non-zero on a parity failure."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2603_05503_b200 import csa, inputs  # noqa: E402
from paper_2603_05503_b200.inputs import Layout  # noqa: E402


def run(lay, heads, masks, rep, order, q, k, v):
    counts = torch.from_numpy(masks.astype(np.uint16).reshape(-1).view(np.int16)).cuda()
    sim = torch.tensor([1.0 if h in rep else 0.0 for h in range(heads)], dtype=torch.float64,
                       device="cuda")
    plan = csa.compile_plan(lay, counts.view(torch.uint16), 1, similarity=sim, anchor_k=5)
    work = csa.build_work_list(plan, 0, heads, order=order)
    out = csa.sparse_attn_fwd(q, k, v, plan, work)
    torch.cuda.synchronize()
    return out


def check(lay, heads, seed, units):
    rng = np.random.default_rng(seed)
    masks = (rng.random((heads, lay.NB, lay.NB)) < 0.4).astype(np.uint8)
    masks[:, np.arange(lay.NB), np.arange(lay.NB)] = 1
    rep = [heads - 1]
    q, k, v = inputs.qkv(1, lay.N, heads, 128, seed=seed, device="cuda")
    single = run(lay, heads, masks, rep, 2, q, k, v)
    pair = run(lay, heads, masks, rep, 3, q, k, v)
    same = torch.equal(single, pair)
    worst = 0.0
    for h, r in units:
        rows = (r * 128, min((r + 1) * 128, lay.N))
        qh, kh, vh = (t[0, :, h].double().cpu().numpy() for t in (q, k, v))
        if h in rep:
            ref, _ = oracle.anchor_attention_rows(lay.F, lay.H, lay.W, qh, kh, vh,
                                                  1 / np.sqrt(128), 5, rows)
        else:
            ref, _ = oracle.masked_attention_rows(qh, kh, vh, 1 / np.sqrt(128), 128, masks[h], rows)
        got = pair[0, rows[0]:rows[1], h].double().cpu().numpy()
        err = np.abs(got - ref)
        worst = max(worst, err.max())
        print(f"  h{h} r{r}: max {err.max():.3e} mean {err.mean():.3e}")
        assert err.max() <= 2e-2 and err.mean() <= 2e-3
    print(f"{lay}: pair == single bitwise: {same}; worst {worst:.3e}")


check(Layout(2, 9, 40, 128), 3, 1, [(0, 0), (1, 5), (2, 2), (0, 3)])
check(Layout(21, 30, 52, 128), 6, 2, [(0, 0), (3, 255), (5, 100), (2, 7)])
print("pair_check OK")
