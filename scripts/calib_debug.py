"""Debug: calibration LSE / E errors vs the oracle for the single-pass, two-pass and lse_in modes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import oracle
from paper_2603_05503_b200 import csa, inputs
from paper_2603_05503_b200.inputs import Layout

for lay, heads, d in [(Layout(2, 5, 25, 64), 2, 64), (Layout(2, 9, 40, 128), 2, 128),
                      (Layout(4, 8, 8, 128), 1, 128)]:
    q, k, _ = inputs.structured_qk(lay, heads, d, 1, 0, alpha=1.0, device="cuda")
    nb = lay.NB
    scale = 1.0 / np.sqrt(d)
    for mode in ("single", "two", "lse_in"):
        counts = torch.zeros(heads * nb * nb, dtype=torch.int16, device="cuda").view(torch.uint16)
        energy = torch.empty(heads * nb * nb, dtype=torch.float32, device="cuda")
        lse_out = torch.empty(heads * lay.N, dtype=torch.float32, device="cuda")
        lse_in = None
        if mode == "lse_in":
            lse_in = torch.from_numpy(np.stack([
                oracle.row_lse(q[0, :, h].double().cpu().numpy(), k[0, :, h].double().cpu().numpy(),
                               scale) for h in range(heads)]).astype(np.float32).reshape(-1)).cuda()
        csa.calib_accumulate(lay, q, k, 0.9, counts, lse_in=lse_in, energy_out=energy,
                             lse_out=lse_out, single_pass=(mode == "single"))
        torch.cuda.synchronize()
        E = energy.view(heads, nb, nb).double().cpu().numpy()
        lg = lse_out.view(heads, lay.N).double().cpu().numpy()
        for h in range(heads):
            qh, kh = q[0, :, h].double().cpu().numpy(), k[0, :, h].double().cpu().numpy()
            ref_lse = oracle.row_lse(qh, kh, scale)
            E_ref = oracle.block_energy(qh, kh, scale, lay.B)
            el = np.abs(lg[h] - ref_lse)
            print(f"{lay} d{d} {mode:6s} h{h} lse err max {el.max():.3e} (argmax row {el.argmax()})"
                  f"  E err {np.abs(E[h] - E_ref).max():.3e}  rowsum-1 {np.abs(E[h].sum(1) - 1).max():.3e}")
            if h == 0 and el.max() > 1e-3:
                print("   lse gpu", lg[h][:8], "\n   lse ref", ref_lse[:8])
