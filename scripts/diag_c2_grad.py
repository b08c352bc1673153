"""Diagnostic (GPU box): per-trajectory C2 gradients of the tensor-core path (gp kernel 1) and the
v0 CUDA-core FFMA path (gp kernel 0), one B = 1 launch per trajectory (bitwise equal to the
full-batch launch, test_batch_invariance_bitwise), saved for comparison with the oracle on the CPU.
    python scripts/diag_c2_grad.py OUTDIR [seed_iterations...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

out = sys.argv[1]
its = [int(a) for a in sys.argv[2:]] or [1]
os.makedirs(out, exist_ok=True)
wl = W.config("C2")
ctx = bagel.setup(wl, device=0)
th = torch.from_numpy(wl.theta).cuda()
for kern in (1, 0):
    ctx.set_gp_kernel(kern)
    for it in its:
        seed = W.rollout_seed(it)
        G = np.zeros((wl.B, wl.n_params), dtype=np.float32)
        cost = np.zeros(wl.B)
        for b in range(wl.B):
            c, g = ctx.rollout_cost_and_grad(th, torch.from_numpy(wl.x0[b:b + 1]).cuda(),
                                             torch.from_numpy(wl.goals[b:b + 1]).cuda(), wl.T, seed, traj_offset=b,
                                             B_global=wl.B)
            G[b] = g.cpu().numpy()
            cost[b] = c
        cf, gf = ctx.rollout_cost_and_grad(th, torch.from_numpy(wl.x0).cuda(), torch.from_numpy(wl.goals).cuda(),
                                           wl.T, seed)
        np.savez_compressed(os.path.join(out, f"grad_k{kern}_it{it}.npz"), G=G, cost=cost, gfull=gf.cpu().numpy(),
                            cfull=cf)
        print(kern, it, "full-batch vs sum of B=1 runs:",
              np.linalg.norm(G.astype(np.float64).sum(0) - gf.cpu().numpy()) / np.linalg.norm(gf.cpu().numpy()),
              flush=True)
