"""Writes tests/golden/c2_fullbatch.npz: the float64 oracle's C2 full-batch cost and gradient (bench
workload: B = 1024, T = 100) for rollout iterations 1..4, with the oracle's own fp32 parity floors
(SURVEY §8(c) item 7): mode 5 = the exponent formed in fp32 exactly as the CUDA kernels form it
(difference first, then the kappa / l scale, FMA-accumulated), mode 1 = every kernel value times
(1 + U(+-2^-22)), three draws.  Calls only oracle/ (and the seeded input generator workloads/).
    python scripts/make_golden_c2.py"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402

wl = W.config("C2")
O.set_num_threads(len(os.sched_getaffinity(0)))
mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
out = {}
for it in (1, 2, 3, 4):
    seed = W.rollout_seed(it)
    ref = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0, wl.goals, wl.T, seed)
    gn = np.linalg.norm(ref["grad"])
    out[f"grad_it{it}"] = ref["grad"]
    out[f"cost_it{it}"] = np.array(ref["cost"])
    p5 = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0, wl.goals, wl.T, seed, perturb_mode=5)
    out[f"floor5_it{it}"] = np.array(np.linalg.norm(p5["grad"] - ref["grad"]) / gn)
    f1 = []
    for ps in (1, 2, 3):
        p1 = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0, wl.goals, wl.T, seed,
                       perturb_mode=1, perturb_seed=ps)
        f1.append(np.linalg.norm(p1["grad"] - ref["grad"]) / gn)
    out[f"floor1_it{it}"] = np.array(f1)
    print(it, ref["cost"], out[f"floor5_it{it}"], f1, flush=True)
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c2_fullbatch.npz"), **out)
