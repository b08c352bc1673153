"""Diagnostic (GPU box): where the C2 full-batch gradient error comes from.  Per-trajectory
gradients of the tensor-core path (gp kernel 1) and the v0 CUDA-core FFMA path (gp kernel 0), one
B = 1 launch per trajectory (bitwise equal to the full-batch launch, test_batch_invariance_bitwise),
against the oracle's per-trajectory gradients, exact and under its fp32-sensitivity perturbations
(mode 1: all kernel values x (1 + U(+-2^-22)), 2: mean path only, 3: variance path only).
    python scripts/diag_c2_grad.py OUT.json [iterations...]"""
import json
import os
import sys
from multiprocessing import Pool

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O  # noqa: E402
import workloads as W  # noqa: E402

wl = W.config("C2")
MDL = None


def _init():
    global MDL
    O.set_num_threads(1)
    MDL = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)


def _oracle_row(args):
    b, seed, mode, ps = args
    r = O.rollout(MDL, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0[b:b + 1], wl.goals[b:b + 1], wl.T, seed,
                  traj_offset=b, B_global=wl.B, perturb_mode=mode, perturb_seed=ps, trace=True)
    return r["grad"], float((r["var"][:, 0, :] / MDL.s[None, :]).min())


def main():
    from paper_2202_13638_b200 import bagel

    out = sys.argv[1]
    its = [int(a) for a in sys.argv[2:]] or [1]
    ctx = bagel.setup(wl, device=0)
    th = torch.from_numpy(wl.theta).cuda()
    res = {}
    pool = Pool(len(os.sched_getaffinity(0)), initializer=_init)
    for it in its:
        seed = W.rollout_seed(it)
        gpu = {}
        for kern in (1, 0):
            ctx.set_gp_kernel(kern)
            G = np.zeros((wl.B, wl.n_params))
            for b in range(wl.B):
                _, g = ctx.rollout_cost_and_grad(th, torch.from_numpy(wl.x0[b:b + 1]).cuda(),
                                                 torch.from_numpy(wl.goals[b:b + 1]).cuda(), wl.T, seed, traj_offset=b,
                                                 B_global=wl.B)
                G[b] = g.double().cpu().numpy()
            gpu[kern] = G
        ctx.set_gp_kernel(1)
        ref = pool.map(_oracle_row, [(b, seed, 0, 0) for b in range(wl.B)])
        Go = np.stack([r[0] for r in ref])
        vmin = np.array([r[1] for r in ref])
        gn = np.linalg.norm(Go.sum(0))
        entry = {"gpu_tc": float(np.linalg.norm(gpu[1].sum(0) - Go.sum(0)) / gn),
                 "gpu_v0": float(np.linalg.norm(gpu[0].sum(0) - Go.sum(0)) / gn)}
        pert = {}
        for mode, ps in ([] if os.environ.get("DIAG_NO_PERTURB") else [(1, 1), (1, 2), (1, 3), (1, 4), (2, 1), (3, 1)]):
            Gp = np.stack([r[0] for r in pool.map(_oracle_row, [(b, seed, mode, ps) for b in range(wl.B)])])
            pert[(mode, ps)] = Gp
            entry[f"floor_m{mode}_s{ps}"] = float(np.linalg.norm(Gp.sum(0) - Go.sum(0)) / gn)
        # per-trajectory error norms (absolute, in units of the batch gradient norm)
        e_tc = np.linalg.norm(gpu[1] - Go, axis=1) / gn
        e_v0 = np.linalg.norm(gpu[0] - Go, axis=1) / gn
        e_p = np.linalg.norm(pert[(1, 1)] - Go, axis=1) / gn if pert else np.zeros(wl.B)
        top = np.argsort(-e_tc)[:15]
        entry["top_rows"] = [{"b": int(b), "err_tc": float(e_tc[b]), "err_v0": float(e_v0[b]), "floor_m1": float(e_p[b]),
                              "floor_m2": float(np.linalg.norm(pert[(2, 1)][b] - Go[b]) / gn) if pert else 0.0,
                              "floor_m3": float(np.linalg.norm(pert[(3, 1)][b] - Go[b]) / gn) if pert else 0.0,
                              "gnorm": float(np.linalg.norm(Go[b]) / gn), "vmin_over_s": float(vmin[b])}
                             for b in top]
        # the batch error without the 10 worst trajectories
        keep = np.ones(wl.B, bool)
        keep[top[:10]] = False
        entry["gpu_tc_without_top10"] = float(np.linalg.norm((gpu[1] - Go)[keep].sum(0)) / gn)
        if pert:
            entry["floor_m1_without_top10"] = float(np.linalg.norm((pert[(1, 1)] - Go)[keep].sum(0)) / gn)
        entry["sum_sq_share_top10_tc"] = float((e_tc[top[:10]] ** 2).sum() / (e_tc ** 2).sum())
        res[it] = entry
        print(json.dumps({it: entry}), flush=True)
    json.dump(res, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
