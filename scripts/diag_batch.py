"""Diagnostic: GPU gradient consistency across batch splits at C2 (B = 1024)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

wl = W.config("C2")
ctx = bagel.setup(wl, device=0)
seed = W.rollout_seed(1)
th = torch.from_numpy(wl.theta).cuda()


def run(off, B, kernel=1):
    ctx.set_gp_kernel(kernel)
    c, g = ctx.rollout_cost_and_grad(th, torch.from_numpy(wl.x0[off:off + B]).cuda(),
                                     torch.from_numpy(wl.goals[off:off + B]).cuda(), wl.T, seed, traj_offset=off,
                                     B_global=wl.B)
    return c, g.double().cpu().numpy().copy()


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


for kernel in (1, 0):
    c_full, g_full = run(0, 1024, kernel)
    for nsh in (2, 4, 8, 16, 64):
        bs = 1024 // nsh
        cs, gs = 0.0, 0
        for i in range(nsh):
            c, g = run(i * bs, bs, kernel)
            cs += c
            gs = gs + g
        print(f"kernel {kernel}: {nsh} shards of {bs}: cost rel {abs(cs - c_full) / abs(c_full):.2e}, "
              f"grad rel {rel(gs, g_full):.2e}", flush=True)
    c2, g2 = run(0, 1024, kernel)
    print(f"kernel {kernel}: repeat full batch: cost {c2 == c_full}, grad identical {np.array_equal(g2, g_full)}")
