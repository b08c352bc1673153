"""Compare the fused (pass 2 + epilogue) and separate epilogue paths on one rollout."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

wl = W.config(sys.argv[1] if len(sys.argv) > 1 else "C2")
B = int(sys.argv[2]) if len(sys.argv) > 2 else wl.B
T = int(sys.argv[3]) if len(sys.argv) > 3 else wl.T
ctx = bagel.setup(wl, device=0)
x0g, gg = W.sample_states_goals(wl.X, wl.p, B)
theta = torch.from_numpy(wl.theta).cuda()
x0 = torch.from_numpy(x0g).cuda()
goals = torch.from_numpy(gg).cuda()
res = {}
for f in ("0", "1"):
    os.environ["BAGEL_P2_EPI"] = f
    tr = ctx.rollout_trace(theta, x0, goals, T, W.rollout_seed(1))
    res[f] = {k: v.cpu().numpy() for k, v in tr.items()}
for k in res["0"]:
    a, b = res["0"][k], res["1"][k]
    d = np.abs(a - b)
    print(k, a.shape, "max diff", d.max(), "first bad", np.argwhere(d > 1e-5)[:6].tolist() if d.max() > 1e-5 else None)
