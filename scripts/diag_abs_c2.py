"""Per-trajectory gradient error of the absolute-target variant at C2 (B = 64, T = 40) against the
oracle and against the oracle's fp32-sensitivity floor (mode 1 and 5)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 40
wl = W.config("C2", target="abs", B=64, T=T)
mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank, abs_target=True)
ctx = bagel.setup(wl, device=0, build_cache=False)
ctx.gp_target_mode(True)
if len(sys.argv) > 2:
    ctx.set_gp_kernel(int(sys.argv[2]))
for m in range(mdl.p):
    ctx.cache_set(m, mdl.alpha[m], mdl.R[m])
seed = W.rollout_seed(8)
th = torch.from_numpy(wl.theta).cuda()
G, R, F1, F5 = [], [], [], []
for b in range(wl.B):
    x0 = torch.from_numpy(wl.x0[b:b + 1]).cuda()
    g = torch.from_numpy(wl.goals[b:b + 1]).cuda()
    _, gg = ctx.rollout_cost_and_grad(th, x0, g, wl.T, seed, traj_offset=b, B_global=wl.B)
    G.append(gg.double().cpu().numpy())
    args = (mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0[b:b + 1], wl.goals[b:b + 1], wl.T, seed)
    R.append(O.rollout(*args, traj_offset=b, B_global=wl.B)["grad"])
    F1.append(O.rollout(*args, traj_offset=b, B_global=wl.B, perturb_mode=1, perturb_seed=1)["grad"])
    F5.append(O.rollout(*args, traj_offset=b, B_global=wl.B, perturb_mode=5, perturb_seed=1)["grad"])
G, R, F1, F5 = map(np.array, (G, R, F1, F5))
tot = np.linalg.norm(R.sum(0))
print("total rel err gpu", np.linalg.norm(G.sum(0) - R.sum(0)) / tot, "floor1", np.linalg.norm(F1.sum(0) - R.sum(0)) / tot,
      "floor5", np.linalg.norm(F5.sum(0) - R.sum(0)) / tot)
e = np.linalg.norm(G - R, axis=1) / tot
f1 = np.linalg.norm(F1 - R, axis=1) / tot
f5 = np.linalg.norm(F5 - R, axis=1) / tot
own = np.linalg.norm(R, axis=1) / tot
for b in np.argsort(-e)[:8]:
    print(f"traj {b}: gpu err {e[b]:.2e}  floor1 {f1[b]:.2e}  floor5 {f5[b]:.2e}  |g_b|/|g| {own[b]:.2e}")
