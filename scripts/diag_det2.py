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
ctx.set_gp_kernel(0)
ref = [t.clone().cpu().numpy() for t in ctx.gp_predict(xs)]
ctx.set_gp_kernel(1)
for rep in range(3):
    out = [t.clone().cpu().numpy() for t in ctx.gp_predict(xs)]
    d = np.abs(out[2] - ref[2]).max(axis=2)  # M x p
    bad = np.argwhere(d > 1e-3 * np.abs(ref[2]).max())
    print("rep", rep, "bad (row, m) count", len(bad), "rows:", sorted(set(bad[:, 0] // 128)), "m:", sorted(set(bad[:, 1])),
          "first", bad[:8].tolist())
    if len(bad):
        r, m = bad[0]
        print("  dmean gpu", out[2][r, m], "v0", ref[2][r, m], "mean", out[0][r, m], ref[0][r, m])
