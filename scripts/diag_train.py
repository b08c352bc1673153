import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import oracle as O, workloads as W
from paper_2202_13638_b200 import bagel
from paper_2202_13638_b200.train import train_policy
wl = W.make_workload(plant="boom", N=500, rank=64, hidden=(256, 256), B=96, T=6)
mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
lo, hi = wl.X[:, :wl.p].min(0), wl.X[:, :wl.p].max(0)
ctx = bagel.setup(wl, device=0)
for m in range(mdl.p):
    ctx.cache_set(m, mdl.alpha[m], mdl.R[m])
for iters in (1, 2, 4):
    th, log = train_policy(ctx, wl.theta, wl.T, iters, wl.B, lo, hi, lr=1e-2, seed0=0x5EED2000)
    th_o, costs_o = O.train(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.T, iters, wl.B, lo, hi, 0x5EED2000, lr=1e-2)
    t = th.cpu().numpy().astype(np.float64)
    d = t - th_o
    big = np.abs(d) > 5e-3
    print(iters, "costs gpu", np.array(log.cost), "or", np.array(costs_o), "rel dtheta", np.linalg.norm(d) / np.linalg.norm(th_o),
          "n(|d|>5e-3)", big.sum(), "max|d|", np.abs(d).max())
# gradient at theta0 on the first iteration's sample
x0 = O.sample_states(0x5EED2000, 0, wl.B, lo, hi, 0).astype(np.float32); g = O.sample_states(0x5EED2000, 0, wl.B, lo, hi, 1).astype(np.float32)
cost, grad = ctx.rollout_cost_and_grad(torch.from_numpy(wl.theta).cuda(), torch.from_numpy(x0).cuda(), torch.from_numpy(g).cuda(), wl.T, 0x5EED2000)
grad = grad.double().cpu().numpy()
ref = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, x0, g, wl.T, 0x5EED2000)
go = ref["grad"]
flip = np.sign(grad) != np.sign(go)
print("grad rel L2", np.linalg.norm(grad - go) / np.linalg.norm(go), "sign flips", flip.sum(), "max |g_o| among flips / max|g_o|", np.abs(go[flip]).max() / np.abs(go).max() if flip.any() else 0)
