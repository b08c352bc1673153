"""C2 full batch (B = 1024, T = 100): GPU cost/gradient vs the oracle, and the oracle's own fp32
floor (sensitivity modes) on the same batch."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

wl = W.config("C2")
seed = W.rollout_seed(1)
t0 = time.time()
mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
args = (mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0, wl.goals, wl.T, seed)
ref = O.rollout(*args)
print(f"oracle full batch in {time.time() - t0:.1f} s", flush=True)
ctx = bagel.setup(wl, device=0)
for kernel in (1, 0):
    ctx.set_gp_kernel(kernel)
    c, g = ctx.rollout_cost_and_grad(torch.from_numpy(wl.theta).cuda(), torch.from_numpy(wl.x0).cuda(),
                                     torch.from_numpy(wl.goals).cuda(), wl.T, seed)
    g = g.double().cpu().numpy()
    print(f"GPU kernel {kernel}: cost rel {abs(c - ref['cost']) / abs(ref['cost']):.2e}  grad rel L2 "
          f"{np.linalg.norm(g - ref['grad']) / np.linalg.norm(ref['grad']):.2e}", flush=True)
for mode, name in ((1, "2^-22 on every kernel value"), (5, "fp32 exponent (diff, then scale)")):
    r = O.rollout(*args, perturb_mode=mode, perturb_seed=1)
    print(f"oracle floor [{name}]: cost rel {abs(r['cost'] - ref['cost']) / abs(ref['cost']):.2e}  grad rel L2 "
          f"{np.linalg.norm(r['grad'] - ref['grad']) / np.linalg.norm(ref['grad']):.2e}", flush=True)
