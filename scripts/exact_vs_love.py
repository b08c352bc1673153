"""LOVE vs exact GP variance on the hot path (the paper's comparison of
BAGEL with "AutoDiff on exact GPs"): Exp. 1 shape (b = 100, H = 300, [8, 8]) on an
N = 700 boom dataset, one rollout_cost_and_grad per measurement, CUDA-event timed; also the largest
LOVE-vs-exact variance gap over the rollout's states (LOVE rank 100 and 256)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 700
wl = W.make_workload(plant="boom", N=N, rank=100, hidden=(8, 8), B=100, T=300, fixed_start=True)
th, x0, g = (torch.from_numpy(a).cuda() for a in (wl.theta, wl.x0, wl.goals))
res = {"N": N, "B": wl.B, "T": wl.T}
traces = {}
for mode in ("love100", "love256", "exact"):
    ctx = bagel.setup(wl, device=0, build_cache=False)
    sec = ctx.exact_cache_build() if mode == "exact" else ctx.love_cache_build(int(mode[4:]))
    grad = torch.empty(ctx.n_params, device="cuda")
    for i in range(3):
        ctx.rollout_cost_and_grad(th, x0, g, wl.T, W.rollout_seed(i), grad=grad)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for i in range(5):
        e0.record()
        cost, _ = ctx.rollout_cost_and_grad(th, x0, g, wl.T, W.rollout_seed(10 + i), grad=grad)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    tr = ctx.rollout_trace(th, x0, g, wl.T, W.rollout_seed(10))
    xs = torch.cat([tr["x"][:-1].reshape(-1, wl.p), torch.zeros(wl.T * wl.B, wl.q, device="cuda")], 1)
    traces[mode] = ctx.gp_predict(xs[: 4096])[1].cpu().numpy()
    res[mode] = {"cache_s": sec, "ms_per_iter": float(np.median(ms)), "cost": cost}
    ctx.close()
for r in ("love100", "love256"):
    res[f"max |v_{r} - v_exact| / s"] = float((np.abs(traces[r] - traces["exact"]) / wl.s).max())
print(json.dumps(res))
