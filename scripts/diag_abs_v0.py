"""Diagnostic (GPU box): absolute targets on the C2 subset of tests/golden/abs_targets.npz,
tensor-core GP step (1) vs v0 FFMA GP step (0), T = 20, 40, 100; and C2 iteration time of both.
    python scripts/diag_abs_v0.py OUTDIR"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

out = sys.argv[1]
os.makedirs(out, exist_ok=True)
wa = W.config("C2", target="abs", B=64, T=100)
ma = O.Model.build(wa.X, wa.Y, wa.ell, wa.s, wa.noise, wa.rank, abs_target=True)
cta = bagel.setup(wa, device=0, build_cache=False)
cta.gp_target_mode(True)
for m in range(wa.p):
    cta.cache_set(m, ma.alpha[m], ma.R[m])
for kern in (1, 0):
    cta.set_gp_kernel(kern)
    for T in (20, 40, 100):
        c, gr = cta.rollout_cost_and_grad(torch.from_numpy(wa.theta).cuda(), torch.from_numpy(wa.x0).cuda(),
                                          torch.from_numpy(wa.goals).cuda(), T, W.rollout_seed(8))
        np.save(os.path.join(out, f"abs_k{kern}_T{T}.npy"), gr.double().cpu().numpy())
wl = W.config("C2")
ctx = bagel.setup(wl, device=0)
th, x0, g = (torch.from_numpy(a).cuda() for a in (wl.theta, wl.x0, wl.goals))
for kern in (1, 0):
    ctx.set_gp_kernel(kern)
    ctx.rollout_cost_and_grad(th, x0, g, wl.T, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for it in range(5):
        ctx.rollout_cost_and_grad(th, x0, g, wl.T, W.rollout_seed(it))
    e1.record()
    torch.cuda.synchronize()
    print(f"gp kernel {kern}: {e0.elapsed_time(e1) / 5:.3f} ms per C2 iteration", flush=True)
