import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import oracle as O, workloads as W
from paper_2202_13638_b200 import bagel
import test_gpu_parity as TP

def run(tag, plant, hidden, B, T, rank, N, abs_t=False, phi="xg", target="delta"):
    wl = W.make_workload(plant=plant, N=N, rank=rank, hidden=hidden, B=B, T=T, phi_mode=phi, target="abs" if abs_t else "delta")
    mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank, abs_target=abs_t)
    ctx = TP._ctx(bagel, wl, build_cache=False)
    if abs_t: ctx.gp_target_mode(True)
    TP._inject(ctx, mdl)
    seed = W.rollout_seed(31)
    cost, grad = TP._rollout_gpu(ctx, wl, wl.goals, seed)
    ref = TP._rollout_oracle(mdl, wl, wl.goals, seed)
    rc = abs(cost - ref["cost"]) / abs(ref["cost"]); rg = np.linalg.norm(grad - ref["grad"]) / np.linalg.norm(ref["grad"])
    print(f"{tag}: cost {rc:.2e} grad {rg:.2e} {'OK' if rc <= 1e-3 and rg <= 1e-3 else 'FAIL'}", flush=True)
    ctx.close()

run("hyd4 wide abs", "hydraulic4", (256, 256), 130, 8, 64, 800, abs_t=True)
run("boom wide abs T40", "boom", (256, 256, 256), 64, 40, 64, 600, abs_t=True)
run("hyd4 wide xgd", "hydraulic4", (200, 136), 70, 5, 96, 900, phi="xgd")
run("boom 7x128 abs", "boom", (128,) * 7, 40, 6, 64, 500, abs_t=True)
run("boom wide rank300", "boom", (256, 256), 200, 5, 300, 1200)
