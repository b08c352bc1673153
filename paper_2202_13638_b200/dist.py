"""Data parallelism over trajectories.

Trajectories are independent given theta and the GP cache (the objective of
Eq.11 is a sum over b) and eps is indexed by the global trajectory
id, so the B trajectories of an iteration are split into contiguous blocks,
one per rank; each rank returns its share of L (already divided by B_global)
and of dL/dtheta, and ONE all_reduce(SUM) of the flat [grad | cost] buffer
finishes the iteration.  With the NCCL process group that collective runs over
NVLink / NVSwitch; the gloo group is used by the CPU tests.
"""
from __future__ import annotations

import torch
import torch.distributed as tdist


def shard(B_global: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous block of rank `rank`: returns (traj_offset, B_local).  Remainders go to the
    lowest ranks so every trajectory is owned exactly once."""
    if B_global < 1 or world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad shard request B={B_global} world={world} rank={rank}")
    base, rem = divmod(B_global, world)
    b_local = base + (1 if rank < rem else 0)
    offset = rank * base + min(rank, rem)
    return offset, b_local


def allreduce_cost_grad(cost: float, grad: torch.Tensor, group=None) -> tuple[float, torch.Tensor]:
    """One all_reduce(SUM) of [grad (|theta|) | cost] in float64 (fixed algorithm -> run-to-run
    reproducible at fixed world size)."""
    if not (tdist.is_available() and tdist.is_initialized()) or tdist.get_world_size(group) == 1:
        return cost, grad
    buf = torch.empty(grad.numel() + 1, dtype=torch.float64, device=grad.device)
    buf[:-1].copy_(grad.reshape(-1))
    buf[-1] = cost
    tdist.all_reduce(buf, op=tdist.ReduceOp.SUM, group=group)
    grad.copy_(buf[:-1].to(grad.dtype).reshape(grad.shape))
    return float(buf[-1].item()), grad


def rollout_cost_and_grad_dp(local_fn, theta, x0_global, goals_global, T: int, seed: int, group=None):
    """Data-parallel iteration.  `local_fn(theta, x0, goals, T, seed, traj_offset, B_global)` returns
    (cost share, grad share) for one contiguous trajectory block -- Context.rollout_cost_and_grad on
    a GPU rank.  Returns the global (L, dL/dtheta) on every rank."""
    world = tdist.get_world_size(group) if tdist.is_initialized() else 1
    rank = tdist.get_rank(group) if tdist.is_initialized() else 0
    B = int(x0_global.shape[0])
    off, bl = shard(B, world, rank)
    cost, grad = local_fn(theta, x0_global[off:off + bl], goals_global[off:off + bl], T, seed, off, B)
    return allreduce_cost_grad(cost, grad, group)


def pin_nccl() -> None:
    """Fix NCCL's algorithm and protocol (SURVEY §8(e) determinism): with them pinned the one
    all_reduce per iteration sums in the same order every run, so results are bitwise repeatable at
    a fixed world size.  Ring + LL: the message is |theta| + 1 doubles (tens of KB, latency bound).
    Call before init_process_group; explicit user settings win."""
    import os

    os.environ.setdefault("NCCL_ALGO", "Ring")
    os.environ.setdefault("NCCL_PROTO", "LL")


def cache_digest(ctx, p: int) -> torch.Tensor:
    """Order-sensitive 64-bit digest of the context's LOVE cache (alpha and R of every output, as raw
    float64 bits), as a 1-element int64 tensor on the context's device."""
    acc = torch.zeros(1, dtype=torch.int64, device=ctx.dev)
    for m in range(p):
        a, R = ctx.cache_get(m)
        for t in (a, R):
            bits = t.contiguous().view(torch.int64).reshape(-1)
            w = torch.arange(1, bits.numel() + 1, device=bits.device, dtype=torch.int64) * 0x9E3779B1
            acc = acc * 1000003 + (bits ^ w).sum().reshape(1)   # int64 arithmetic wraps
    return acc


def verify_replicated_cache(ctx, p: int, group=None) -> None:
    """Each rank builds the replicated LOVE cache itself (deterministic fixed-order fp64 build); check
    that every rank's copy is bit-identical (min == max of the digest over ranks), else raise."""
    if not (tdist.is_available() and tdist.is_initialized()) or tdist.get_world_size(group) == 1:
        return
    d = cache_digest(ctx, p)
    lo, hi = d.clone(), d.clone()
    tdist.all_reduce(lo, op=tdist.ReduceOp.MIN, group=group)
    tdist.all_reduce(hi, op=tdist.ReduceOp.MAX, group=group)
    if int(lo.item()) != int(hi.item()):
        raise RuntimeError("LOVE caches differ across ranks (non-deterministic cache build)")
