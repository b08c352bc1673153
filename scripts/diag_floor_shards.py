"""Where does the C2 full-batch gradient sensitivity come from?  Oracle exact vs 2^-22-perturbed,
per shard of 64 trajectories, then per trajectory inside the worst shard."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402

wl = W.config("C2")
seed = W.rollout_seed(1)
mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)


def run(off, n, mode):
    return O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0[off:off + n], wl.goals[off:off + n], wl.T,
                     seed, traj_offset=off, B_global=wl.B, perturb_mode=mode, perturb_seed=1)


gtot = None
rows = []
for off in range(0, 1024, 64):
    a, b = run(off, 64, 0), run(off, 64, 1)
    gtot = a["grad"] if gtot is None else gtot + a["grad"]
    rows.append((np.linalg.norm(b["grad"] - a["grad"]), off, np.linalg.norm(a["grad"])))
tot = np.linalg.norm(gtot)
rows.sort(reverse=True)
print("total |grad| =", tot)
for d, off, gn in rows[:6]:
    print(f"shard {off:4d}: |d grad| = {d:.3e} ({d / tot:.2e} of |grad|), |grad shard| = {gn:.3e}")
worst = rows[0][1]
per = []
for b in range(worst, worst + 64):
    a, p = run(b, 1, 0), run(b, 1, 1)
    per.append((np.linalg.norm(p["grad"] - a["grad"]), b, np.linalg.norm(a["grad"]), a["ret"][0]))
per.sort(reverse=True)
for d, b, gn, ret in per[:8]:
    print(f"  traj {b}: |d grad| = {d:.3e} ({d / tot:.2e} of |grad|), |grad_b| = {gn:.3e}, return {ret:.3f}")
