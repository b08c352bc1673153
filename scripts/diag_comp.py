"""Diagnostic (GPU box): Kahan-compensated mean columns (BAGEL_P1_COMPENSATED) -- C2 step time and
full-batch gradients (4 iterations) and the absolute-target subset (T = 20, 40, 100), saved for
comparison with tests/golden/*.npz.   python scripts/diag_comp.py OUTDIR"""
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
wl = W.config("C2")
th, x0, g = (torch.from_numpy(a).cuda() for a in (wl.theta, wl.x0, wl.goals))
wa = W.config("C2", target="abs", B=64, T=100)
ma = O.Model.build(wa.X, wa.Y, wa.ell, wa.s, wa.noise, wa.rank, abs_target=True)
for comp in ("0", "1"):
    os.environ["BAGEL_P1_COMPENSATED"] = comp
    ctx = bagel.setup(wl, device=0)
    for it in (1, 2, 3, 4):
        c, gr = ctx.rollout_cost_and_grad(th, x0, g, wl.T, W.rollout_seed(it))
        np.save(os.path.join(out, f"g_c{comp}_it{it}.npy"), gr.double().cpu().numpy())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for it in range(10):
        ctx.rollout_cost_and_grad(th, x0, g, wl.T, W.rollout_seed(it))
    e1.record()
    torch.cuda.synchronize()
    print(f"compensated {comp}: {e0.elapsed_time(e1) / 10:.3f} ms per C2 iteration", flush=True)
    ctx.close()
    cta = bagel.setup(wa, device=0, build_cache=False)
    cta.gp_target_mode(True)
    for m in range(wa.p):
        cta.cache_set(m, ma.alpha[m], ma.R[m])
    for T in (20, 40, 100):
        c, gr = cta.rollout_cost_and_grad(torch.from_numpy(wa.theta).cuda(), torch.from_numpy(wa.x0).cuda(),
                                          torch.from_numpy(wa.goals).cuda(), T, W.rollout_seed(8))
        np.save(os.path.join(out, f"abs_c{comp}_T{T}.npy"), gr.double().cpu().numpy())
    cta.close()
