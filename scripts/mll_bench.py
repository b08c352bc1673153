"""Time gp_log_marginal_likelihood (value + gradient, fp64) at the configs' dataset sizes and report
the fp64 FMA roofline fraction: algorithmic flops ~ N^3/3 (Cholesky) + N^3/3 (triangular inverse)
+ N^3/3 (Khat^-1 tiles) = N^3, against the B200 fp64 peak (B200_PROFILING.md)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402
from paper_2202_13638_b200.fit import fit_hyperparameters  # noqa: E402

out = []
for cfg in (sys.argv[1:] or ["E1", "C2", "C4"]):
    wl = W.config(cfg, B=1)
    ctx = bagel.Context(0)
    ctx.gp_load(wl.X, wl.Y, wl.ell, wl.s, wl.noise)
    ctx.log_marginal_likelihood(0)  # warm-up / workspace
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        v, g = ctx.log_marginal_likelihood(0)
        ts.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    v1, _ = ctx.log_marginal_likelihood(0, want_grad=False)
    t_val = time.perf_counter() - t0
    rec = {"config": cfg, "N": wl.N, "d": wl.d, "mll": v, "s_value_and_grad": float(np.median(ts)),
           "s_value_only": t_val, "gflops_fp64": wl.N ** 3 / np.median(ts) / 1e9}
    if wl.N <= 5000:
        t0 = time.perf_counter()
        phi, log = fit_hyperparameters(ctx, 0, iters=100, lr=0.05)
        rec.update(fit_100_steps_s=time.perf_counter() - t0, fit_mll_start=log.mll[0], fit_mll_end=log.mll[-1],
                   fit_steps=log.steps)
    out.append(rec)
    print(json.dumps(rec), flush=True)
    ctx.close()
