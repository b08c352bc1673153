"""Run the GP step (pass 1 [+ fused reduce 1], pass 2) a few times at the bench shape (for ncu)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

wl = W.config(sys.argv[1] if len(sys.argv) > 1 else "C2")
ctx = bagel.setup(wl, device=0)
xs = torch.from_numpy(np.random.default_rng(0).uniform(-1.5, 1.5, (wl.B, wl.d)).astype(np.float32)).cuda()
for _ in range(4):
    ctx.gp_predict(xs)
torch.cuda.synchronize()
print("ok")
