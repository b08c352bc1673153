"""Per-CTA event timelines of the tensor-core GP kernels at the bench shape (C2, B = 1024)."""
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
for _ in range(3):
    ctx.gp_predict(xs)
ctx.debug_trace(True)
ctx.gp_predict(xs)
for which, name, ev in ((4, "pass1", ["start", "first MMA commit", "last MMA issued", "generators done", "done wait",
                                      "end", "grid barrier", "reduce done", "tile copied", "w0 loads summed", "w0 row totals"]),
                        (5, "pass2", ["start", "zready (MMA)", "tile0 MMAs issued", "all MMAs issued", "epilogue done",
                                      "end", "zready (epi)", "setup done", "Z loads returned"])):
    st = ctx.debug_stamps(which).astype(np.int64)
    used = st[:, 0] > 0
    st = st[used]
    t0 = st[:, 0].min()
    print(f"{name}: {used.sum()} CTAs, kernel span {(st.max() - t0) / 1e3:.2f} us")
    for k, e in enumerate(ev):
        v = (st[:, k] - t0) / 1e3
        v = v[st[:, k] > 0]
        if len(v):
            print(f"   {e:22s} min {v.min():7.2f}  median {np.median(v):7.2f}  max {v.max():7.2f} us")
