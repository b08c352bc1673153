import sys, os
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
import oracle as O, workloads as W
from paper_2202_13638_b200 import bagel
import test_gpu_parity as TP
hidden = tuple(int(x) for x in sys.argv[1].split(","))
wl = W.make_workload(plant="boom", N=600, rank=64, hidden=hidden, B=200, T=4)
mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
ctx = TP._ctx(bagel, wl, build_cache=False)
TP._inject(ctx, mdl)
goals = (wl.x0 + np.array([0.3, -0.1], dtype=np.float32)).astype(np.float32)
seed = W.rollout_seed(12)
cost, grad = TP._rollout_gpu(ctx, wl, goals, seed)
ref = TP._rollout_oracle(mdl, wl, goals, seed)
g0 = ref["grad"]
off = 0
sz = wl.sizes
print("sizes", sz, "cost rel", abs(cost - ref["cost"]) / abs(ref["cost"]))
for l in range(len(sz) - 1):
    i, o = sz[l], sz[l + 1]
    W_ = slice(off, off + i * o); b_ = slice(off + i * o, off + i * o + o)
    for nm, sl in (("W", W_), ("b", b_)):
        e = np.linalg.norm(grad[sl] - g0[sl]) / max(np.linalg.norm(g0[sl]), 1e-30)
        print(f"layer {l} {nm} ({o}x{i}) rel {e:.2e}  |g| {np.linalg.norm(g0[sl]):.3e}  nan {np.isnan(grad[sl]).sum()}")
    off += i * o + o
