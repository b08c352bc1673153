"""In-kernel timelines of the GP-step kernels (k_p1_tc stamps in debug buffer 4, k_p2_tc in 5; %globaltimer,
16 slots per CTA) for the last step of a rollout at a config: per slot, min / median / max over CTAs,
relative to the earliest CTA start.  python scripts/gp_trace.py C2 [T]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 10
wl = W.config(name, T=T)
ctx = bagel.setup(wl, device=0)
th = torch.from_numpy(wl.theta).cuda()
x0 = torch.from_numpy(wl.x0).cuda()
g = torch.from_numpy(wl.goals).cuda()
ctx.rollout_cost_and_grad(th, x0, g, T, 1)
ctx.debug_trace(True)
ctx.rollout_cost_and_grad(th, x0, g, T, 1)
torch.cuda.synchronize()
for which, kern in ((4, "k_p1_tc"), (5, "k_p2_tc")):
    st = ctx.debug_stamps(which)[:3000].astype(np.int64)  # [cta][16]
    rows = st[st[:, 0] > 0]
    if len(rows) == 0:
        continue
    t0 = rows[:, 0].min()
    print(f"{kern}: {len(rows)} CTAs")
    for k in range(16):
        col = rows[:, k]
        col = col[col > 0]
        if len(col):
            r = (col - t0) / 1000.0
            print(f"  slot {k:2d}: n {len(col):4d}  min {r.min():8.2f}  med {np.median(r):8.2f}  max {r.max():8.2f} us")
