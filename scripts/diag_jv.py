"""Diagnostic (GPU box): GP moments and input Jacobians along the C2 trajectories whose gradients
carry the tensor-core path's error (scripts/diag_c2_grad.py), tensor-core kernels (1) vs v0 FFMA (0)
vs the oracle: relative errors of mu, v, J^mu, J^v and of the reverse-pass input A = J^mu + f J^v.
    python scripts/diag_jv.py OUT.json"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

wl = W.config("C2")
mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
ctxs = {mt: bagel.setup(wl, device=0) for mt in ("default", "6", "2")}
ctx = ctxs["default"]
res = {}
for it, rows in [(1, [240, 206, 766, 178, 5, 10, 11]), (2, [240, 727, 697, 12])]:
    seed = W.rollout_seed(it)
    for b in rows:
        tr = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0[b:b + 1], wl.goals[b:b + 1], wl.T, seed,
                       traj_offset=b, B_global=1, trace=True)
        x = tr["x"][:-1, 0, :]
        u = O.policy_act(wl.sizes, "xg", wl.theta, x, np.repeat(wl.goals[b:b + 1].astype(np.float64), wl.T, 0))
        xs = np.concatenate([x, u], 1).astype(np.float32)
        om, ov, ojm, ojv, mb, vb = mdl.predict(xs.astype(np.float64))
        eps = np.array([[O.rollout_eps(seed, b, t, m) for m in range(wl.p)] for t in range(wl.T)])
        f = eps / (2 * np.sqrt(np.maximum(ov, 1e-12)))
        oA = ojm + f[:, :, None] * ojv
        entry = {}
        for kern in ("1", "0", "1_mt6", "1_mt2"):
            mt = kern[4:] if "mt" in kern else "default"
            cx = ctxs[mt]
            cx.set_gp_kernel(int(kern[0]))
            if mt != "default":   # the split is chosen when the workspace is (re)built, i.e. on this call
                os.environ["BAGEL_P1_MAX_TILES"] = mt
            gm, gv, gjm, gjv = [t.double().cpu().numpy() for t in cx.gp_predict(torch.from_numpy(xs).cuda())]
            os.environ.pop("BAGEL_P1_MAX_TILES", None)
            cx.set_gp_kernel(1)
            gA = gjm + f[:, :, None] * gjv

            def rel(a, r):
                return float(np.median(np.linalg.norm(a - r, axis=-1) / np.maximum(np.linalg.norm(r, axis=-1), 1e-30)))

            def relmax(a, r):
                return float(np.max(np.linalg.norm(a - r, axis=-1) / np.maximum(np.linalg.norm(r, axis=-1), 1e-30)))

            entry[f"k{kern}"] = {"mu_abs_med": float(np.median(np.abs(gm - om))), "mu_abs_max": float(np.max(np.abs(gm - om))),
                                 "v_rel_med": float(np.median(np.abs(gv - ov) / ov)), "v_rel_max": float(np.max(np.abs(gv - ov) / ov)),
                                 "jmu_rel_med": rel(gjm, ojm), "jmu_rel_max": relmax(gjm, ojm),
                                 "jv_rel_med": rel(gjv, ojv), "jv_rel_max": relmax(gjv, ojv),
                                 "A_rel_med": rel(gA, oA), "A_rel_max": relmax(gA, oA)}
        entry["v_over_s_min"] = float((ov / wl.s[None, :]).min())
        entry["fJv_over_Jmu_med"] = float(np.median(np.linalg.norm(f[:, :, None] * ojv, axis=-1) /
                                                    np.linalg.norm(ojm, axis=-1)))
        res[f"it{it}_b{b}"] = entry
        print(f"it{it}_b{b}", json.dumps(entry), flush=True)
json.dump(res, open(sys.argv[1], "w"), indent=1)
