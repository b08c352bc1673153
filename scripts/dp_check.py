"""Multi-GPU data-parallel check (run under torchrun, one rank per GPU, NCCL): every rank builds the
replicated LOVE cache (checked bit-identical across ranks), rolls out its contiguous block of the
global batch (strong scaling), one all_reduce of [grad | cost]; rank 0 then recomputes the whole
batch on its own GPU and compares.  Per-trajectory arithmetic is batch-invariant (N-only split
boundaries), so the shards replay the single-GPU trajectories bit for bit and only the order of the
final theta-gradient sums differs.  Prints one JSON line on rank 0; exit code 1 on a mismatch.
    torchrun --nproc-per-node 2 scripts/dp_check.py [CONFIG]"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as tdist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402
from paper_2202_13638_b200.dist import allreduce_cost_grad, pin_nccl, shard, verify_replicated_cache  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
rank, world, local = (int(os.environ.get(k, d)) for k, d in (("RANK", 0), ("WORLD_SIZE", 1), ("LOCAL_RANK", 0)))
torch.cuda.set_device(local)
pin_nccl()
tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
wl = W.config(name)
ctx = bagel.setup(wl, device=local)
verify_replicated_cache(ctx, wl.p)
off, bl = shard(wl.B, world, rank)
th = torch.from_numpy(wl.theta).cuda()
seed = W.rollout_seed(1)
cost, grad = ctx.rollout_cost_and_grad(th, torch.from_numpy(wl.x0[off:off + bl]).cuda(),
                                       torch.from_numpy(wl.goals[off:off + bl]).cuda(), wl.T, seed, traj_offset=off,
                                       B_global=wl.B)
cost, grad = allreduce_cost_grad(cost, grad)
# the same iteration again: bitwise repeatable with NCCL's algorithm and protocol pinned
cost2, grad2 = ctx.rollout_cost_and_grad(th, torch.from_numpy(wl.x0[off:off + bl]).cuda(),
                                         torch.from_numpy(wl.goals[off:off + bl]).cuda(), wl.T, seed, traj_offset=off,
                                         B_global=wl.B)
cost2, grad2 = allreduce_cost_grad(cost2, grad2)
ok = True
out = {"config": name, "world": world}
if rank == 0:
    c1, g1 = ctx.rollout_cost_and_grad(th, torch.from_numpy(wl.x0).cuda(), torch.from_numpy(wl.goals).cuda(), wl.T,
                                       seed)
    g, gr, gs = (t.double().cpu().numpy() for t in (grad, grad2, g1))
    out.update(cost_rel=abs(cost - c1) / abs(c1), grad_rel=float(np.linalg.norm(g - gs) / np.linalg.norm(gs)),
               repeat_bitwise=bool(cost == cost2 and np.array_equal(g, gr)))
    ok = out["cost_rel"] <= 1e-6 and out["grad_rel"] <= 1e-6 and out["repeat_bitwise"]
    out["ok"] = ok
    print(json.dumps(out), flush=True)
tdist.destroy_process_group()
sys.exit(0 if ok else 1)
