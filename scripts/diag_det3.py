import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W
from paper_2202_13638_b200 import bagel
wl = W.config("C2")
ctx = bagel.setup(wl, device=0)
rng = np.random.default_rng(0)
M = 2048
xs = torch.from_numpy(rng.uniform(-1.5, 1.5, (M, 3)).astype(np.float32)).cuda()
ctx.gp_predict(xs)
S1 = 4
n = S1 * 2 * M * 4
ref = ctx.debug_buffer(0, n).reshape(S1, 2, M, 4)
for rep in range(6):
    ctx.gp_predict(xs)
    h = ctx.debug_buffer(0, n).reshape(S1, 2, M, 4)
    diff = np.argwhere(h != ref)
    if len(diff):
        s_, m_, r_, c_ = diff.T
        print("rep", rep, "P1h differs:", len(diff), "splits", sorted(set(s_)), "m", sorted(set(m_)), "cols", sorted(set(c_)),
              "row groups(32)", sorted(set(r_ // 32))[:10], "rows mod 128 groups", sorted(set((r_ % 128) // 32)))
        i = tuple(diff[0]); print("  e.g.", i, h[i], ref[i])
    else:
        print("rep", rep, "P1h identical")
