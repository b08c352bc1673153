"""Diagnostic (GPU box): per-trajectory gradient error of the CUDA path vs the oracle at C2,
with each trajectory's minimum LOVE variance / s and how far it strays from the data box."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
wl = W.config("C2")
mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
ctx = bagel.setup(wl, device=0)
seed = W.rollout_seed(1)
tr = ctx.rollout_trace(wl.theta, wl.x0, wl.goals, wl.T, seed)
var = tr["var"].double().cpu().numpy()  # T x B x p
x = tr["x"].double().cpu().numpy()
lo, hi = wl.X[:, :2].min(0), wl.X[:, :2].max(0)
rows = []
gsum_g = np.zeros(wl.n_params)
gsum_o = np.zeros(wl.n_params)
for b in range(n):
    c, g = ctx.rollout_cost_and_grad(torch.from_numpy(wl.theta).cuda(), torch.from_numpy(wl.x0[b:b + 1]).cuda(),
                                     torch.from_numpy(wl.goals[b:b + 1]).cuda(), wl.T, seed, traj_offset=b,
                                     B_global=wl.B)
    g = g.double().cpu().numpy()
    ref = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0[b:b + 1], wl.goals[b:b + 1], wl.T,
                    seed, traj_offset=b, B_global=wl.B)
    gsum_g += g
    gsum_o += ref["grad"]
    out = np.maximum(0, np.maximum(lo - x[:, b], x[:, b] - hi)).max()
    rows.append((np.linalg.norm(g - ref["grad"]), np.linalg.norm(ref["grad"]), abs(c - ref["cost"]) / abs(ref["cost"]),
                 (var[:, b] / wl.s).min(), out, b))
rows.sort(reverse=True)
print("abs_err  |g_b|  cost_rel  min(v/s)  out_of_box  b")
for r in rows[:15]:
    print("%.3e %.3e %.2e %.2e %.3f %d" % r)
print("sum over %d trajectories: grad rel L2 = %.3e" % (n, np.linalg.norm(gsum_g - gsum_o) / np.linalg.norm(gsum_o)))
print("global min v/s over batch:", (var / wl.s).min(), " fraction of (t,b,m) with v/s < 1e-4:",
      np.mean(var / wl.s < 1e-4))
