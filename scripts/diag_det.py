"""Diagnostic: bitwise determinism of gp_predict (tc path) vs batch size."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

wl = W.config("C2")
ctx = bagel.setup(wl, device=0)
rng = np.random.default_rng(0)
for M in (128, 256, 512, 640, 768, 896, 1024, 2048):
    xs = torch.from_numpy(rng.uniform(-1.5, 1.5, (M, 3)).astype(np.float32)).cuda()
    outs = [[t.clone() for t in ctx.gp_predict(xs)] for _ in range(4)]
    same = [all(torch.equal(outs[0][i], o[i]) for o in outs[1:]) for i in range(4)]
    ctx.set_gp_kernel(0)
    ref = ctx.gp_predict(xs)
    ctx.set_gp_kernel(1)
    err = [float(((outs[0][i] - ref[i]).abs().max() / ref[i].abs().max()).item()) for i in range(4)]
    print(f"M={M}: deterministic mean/var/dmean/dvar {same}; max rel diff vs v0 {['%.1e' % e for e in err]}",
          flush=True)
