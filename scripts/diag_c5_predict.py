"""C5: GP moments of the same 160 query points computed in a small launch (fused, split-K) and as
the first rows of a 65,536-row launch (the rollout's unsplit multi-wave shape), both against the
oracle on the GPU-built cache."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
wl = W.config(name, T=3)
ctx = bagel.setup(wl, device=0)
mdl = O.Model(wl.X, wl.ell, wl.s, *[np.stack(a) for a in zip(*[(x.cpu().numpy(), r.cpu().numpy()) for x, r in
                                                              (ctx.cache_get(m) for m in range(wl.p))])])
rng = np.random.default_rng(1)
xs = np.concatenate([wl.X[rng.integers(0, wl.N, 96)] + rng.normal(0, 0.05, (96, wl.d)),
                     rng.uniform(-2.0, 2.0, (64, wl.d))]).astype(np.float32)
big = np.concatenate([xs, rng.uniform(-2, 2, (wl.B - len(xs), wl.d)).astype(np.float32)])
om, ov, ojm, ojv, mb, vb = mdl.predict(xs.astype(np.float64))
U = 2.0 ** -24
for tag, arr in (("small launch", xs), ("B-row launch", big)):
    mean, var, dm, dv = [t[: len(xs)].double().cpu().numpy() for t in ctx.gp_predict(torch.from_numpy(arr).cuda())]
    em = np.abs(mean - om) / (32 * U * mb)
    ev = np.abs(var - ov) / (32 * U * vb)
    print(f"{tag}: mean err/cond-term max {em.max():.3g} median {np.median(em):.3g}; "
          f"var err/cond-term max {ev.max():.3g}; max |dmu| {np.abs(mean - om).max():.3g}, max |dv|/s {(np.abs(var - ov) / wl.s).max():.3g}; "
          f"max |dJmu| {np.abs(dm - ojm).max():.3g}")
