"""Times one BBMM evaluation (gp_log_marginal_likelihood_bbmm) at a workload's N through the C ABI,
with a per-kernel breakdown when run under ncu's launch list.  Usage: bbmm_prof.py C4 8 100"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
t = int(sys.argv[2]) if len(sys.argv) > 2 else 8
J = int(sys.argv[3]) if len(sys.argv) > 3 else 100
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
wl = W.config(name)
ctx = bagel.Context(0)
ctx.gp_load(wl.X, wl.Y, wl.ell, wl.s, wl.noise)
h = ctx.loaded_log_hyp(0)
for r in range(reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    v, g, ld = ctx.log_marginal_likelihood_bbmm(0, h, t, J, 0, want_grad=True)
    tg = time.perf_counter() - t0
    t0 = time.perf_counter()
    v2, _, _ = ctx.log_marginal_likelihood_bbmm(0, h, t, J, 0, want_grad=False)
    tn = time.perf_counter() - t0
    print(f"{name} N={wl.X.shape[0]} t={t} J={J}: with grad {tg * 1e3:.1f} ms, no grad {tn * 1e3:.1f} ms, "
          f"mll {v:.6e} logdet {ld:.6e}", flush=True)
ctx.close()
