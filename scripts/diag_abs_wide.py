import sys, os; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import oracle as O, workloads as W
from paper_2202_13638_b200 import bagel
import test_gpu_parity as TP
wl = W.make_workload(plant="boom", N=600, rank=64, hidden=(256, 256, 256), B=64, T=40, target="abs")
mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank, abs_target=True)
ctx = TP._ctx(bagel, wl, build_cache=False)
ctx.gp_target_mode(True)
TP._inject(ctx, mdl)
seed = W.rollout_seed(31)
cost, grad = TP._rollout_gpu(ctx, wl, wl.goals, seed)
ref = TP._rollout_oracle(mdl, wl, wl.goals, seed)
g0 = ref["grad"]; n0 = np.linalg.norm(g0)
print("MLP_TC", os.environ.get("BAGEL_MLP_TC", "1"), "grad rel", np.linalg.norm(grad - g0) / n0, flush=True)
if os.environ.get("ENV"):
    for ps in range(4):
        r = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0, wl.goals, wl.T, seed, B_global=wl.B, perturb_mode=1, perturb_seed=ps)
        print("oracle envelope mode1 seed", ps, np.linalg.norm(r["grad"] - g0) / n0, flush=True)
