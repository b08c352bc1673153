"""Timeline of the step epilogue kernel (t = 50) inside one rollout at the bench shape."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

wl = W.config(sys.argv[1] if len(sys.argv) > 1 else "C2")
ctx = bagel.setup(wl, device=0)
x0g, gg = W.sample_states_goals(wl.X, wl.p, wl.B)
theta = torch.from_numpy(wl.theta).cuda()
x0 = torch.from_numpy(x0g).cuda()
goals = torch.from_numpy(gg).cuda()
grad = torch.empty(ctx.n_params, device="cuda")
for i in range(3):
    ctx.rollout_cost_and_grad(theta, x0, goals, wl.T, W.rollout_seed(i), traj_offset=0, B_global=wl.B, grad=grad)
ctx.debug_trace(True)
ctx.rollout_cost_and_grad(theta, x0, goals, wl.T, W.rollout_seed(9), traj_offset=0, B_global=wl.B, grad=grad)
torch.cuda.synchronize()
names = ["start", "theta staged", "P2 sums", "x', reward", "policy", "end"]
allst = {}
for which, nm in ((6, "epilogue"), (4, "pass1"), (5, "pass2")):
    st = ctx.debug_stamps(which).astype(np.int64)
    st = st[st[:, 0] > 0]
    if not len(st):
        continue
    t0 = st[:, 0].min()
    allst[nm] = (st[:, 0].min(), st[st > 0].max())
    print(f"{nm}: {len(st)} CTAs, span {(st[st > 0].max() - t0) / 1e3:.2f} us")
    for k in range(16):
        v = st[:, k]
        v = v[v > 0]
        if len(v):
            v = (v - t0) / 1e3
            print(f"   [{k:2d}] {names[k] if nm == 'epilogue' and k < len(names) else '':14s} min {v.min():7.2f}  "
                  f"median {np.median(v):7.2f}  max {v.max():7.2f} us")

a0, a1 = allst["pass1"]
b0, b1 = allst["pass2"]
s1 = ctx.debug_stamps(4).astype(np.int64)
s2 = ctx.debug_stamps(5).astype(np.int64)
s1 = s1[s1[:, 0] > 0]
s2 = s2[s2[:, 0] > 0]
p1_end = s1[:, 7].max()
print(f"last step: pass1 last CTA done -> pass2 median Z loads returned: {(np.median(s2[:, 8]) - p1_end) / 1e3:.2f} us, "
      f"-> pass2 median zready: {(np.median(s2[:, 6]) - p1_end) / 1e3:.2f} us, -> pass2 median start {(np.median(s2[:, 0]) - p1_end) / 1e3:.2f} us")
if "epilogue" in allst:
    e0, e1 = allst["epilogue"]
    print(f"epilogue(T-2) end -> pass1(T-1) start: {(a0 - e1) / 1e3:.2f} us")
