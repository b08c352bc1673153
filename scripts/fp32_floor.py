"""fp32 parity floor of the C2 rollout (oracle sensitivity mode):
relative change of the cost and gradient when every kernel value carries a 2^-22 relative
perturbation (all / mean path only / variance path only)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
off = int(sys.argv[2]) if len(sys.argv) > 2 else 0
wl = W.config("C2")
mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
seed = W.rollout_seed(1)
args = (mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0[off:off + n], wl.goals[off:off + n], wl.T, seed)
base = O.rollout(*args, traj_offset=off, B_global=wl.B)
modes = [(1, "all kernel values"), (2, "mean path only"), (3, "variance path only"),
         (4, "fp32 exponent (scale, then diff)"), (5, "fp32 exponent (diff, then scale)")]
for mode, name in modes:
    for ps in ((1, 2) if mode < 4 else (0,)):
        r = O.rollout(*args, traj_offset=off, B_global=wl.B, perturb_mode=mode, perturb_seed=ps)
        dc = abs(r["cost"] - base["cost"]) / abs(base["cost"])
        dg = np.linalg.norm(r["grad"] - base["grad"]) / np.linalg.norm(base["grad"])
        print(f"{n} trajectories from {off}, perturb {name:20s} seed {ps}: cost rel {dc:.2e}  grad rel L2 {dg:.2e}",
              flush=True)
