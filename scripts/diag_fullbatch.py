"""Diagnostic (GPU box): C2 full-batch gradients (bench launch shape) of the tensor-core path and the
v0 FFMA path for a few rollout iterations, saved for comparison with oracle references on the CPU.
    python scripts/diag_fullbatch.py OUTDIR it1 [it2 ...]"""
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
ctx = bagel.setup(wl, device=0)
th, x0, g = (torch.from_numpy(a).cuda() for a in (wl.theta, wl.x0, wl.goals))
for it in map(int, sys.argv[2:]):
    for kern in (1, 0):
        ctx.set_gp_kernel(kern)
        c, gr = ctx.rollout_cost_and_grad(th, x0, g, wl.T, W.rollout_seed(it))
        np.save(os.path.join(out, f"g_it{it}_k{kern}.npy"), gr.double().cpu().numpy())
        print(it, kern, c, flush=True)
    ctx.set_gp_kernel(1)
