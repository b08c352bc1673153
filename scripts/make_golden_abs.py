"""Writes tests/golden/abs_targets.npz: the float64 oracle's cost and gradient for the absolute-target
variant ("y = x_{k+1}", NEXT-4) on C2's data and policy, a 64-trajectory block, horizons
T = 20, 40, 100, with the oracle's own fp32 parity floors (mode 5 = the exponent
formed in fp32 as the CUDA kernels form it; mode 1 = kernel values x (1 + U(+-2^-22)), three draws).
Calls only oracle/ and the seeded input generator.   python scripts/make_golden_abs.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402

O.set_num_threads(len(os.sched_getaffinity(0)))
out = {}
wl = W.config("C2", target="abs", B=64, T=100)
mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank, abs_target=True)
seed = W.rollout_seed(8)
for T in (20, 40, 100):
    ref = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0, wl.goals, T, seed)
    gn = np.linalg.norm(ref["grad"])
    out[f"grad_T{T}"] = ref["grad"]
    out[f"cost_T{T}"] = np.array(ref["cost"])
    floors = []
    for mode, ps in ((5, 0), (1, 1), (1, 2), (1, 3)):
        p = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0, wl.goals, T, seed,
                      perturb_mode=mode, perturb_seed=ps)
        floors.append(np.linalg.norm(p["grad"] - ref["grad"]) / gn)
    out[f"floors_T{T}"] = np.array(floors)
    print(T, ref["cost"], floors, flush=True)
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "abs_targets.npz"), **out)
