"""Diagnostic (GPU box): the tensor-core accumulation-chain length (tiles of 32 training points per
TMEM accumulator chain, BAGEL_P1_MAX_TILES) against C2 full-batch gradient parity and step time.
    python scripts/diag_chain.py OUTDIR max_tiles..."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

out = sys.argv[1]
os.makedirs(out, exist_ok=True)
wl = W.config("C2")
th, x0, g = (torch.from_numpy(a).cuda() for a in (wl.theta, wl.x0, wl.goals))
for mt in sys.argv[2:]:
    os.environ["BAGEL_P1_MAX_TILES"] = mt
    ctx = bagel.setup(wl, device=0)
    for it in (1, 2, 3, 4):
        c, gr = ctx.rollout_cost_and_grad(th, x0, g, wl.T, W.rollout_seed(it))
        np.save(os.path.join(out, f"g_mt{mt}_it{it}.npy"), gr.double().cpu().numpy())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for it in range(10):
        ctx.rollout_cost_and_grad(th, x0, g, wl.T, W.rollout_seed(it))
    e1.record()
    torch.cuda.synchronize()
    print(f"max_tiles {mt}: {e0.elapsed_time(e1) / 10:.3f} ms per iteration", flush=True)
    ctx.close()
