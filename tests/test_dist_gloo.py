"""Multi-rank data parallelism on CPU (gloo, world_size 2): sharding arithmetic and the
single [grad | cost] all_reduce reproduce the unsharded iteration.  The per-rank compute
here is the oracle (this test covers the host-side logic; the GPU kernels are covered by
the -m gpu parity tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

from paper_2202_13638_b200.dist import allreduce_cost_grad, rollout_cost_and_grad_dp, shard


@pytest.mark.parametrize("B,world", [(1, 1), (7, 2), (8, 2), (1024, 8), (65536, 8), (13, 4), (3, 8)])
def test_shard_partitions_exactly(B, world):
    if world > B:
        # more ranks than trajectories: the empty ranks own nothing
        blocks = [shard(B, world, r) for r in range(world)]
    else:
        blocks = [shard(B, world, r) for r in range(world)]
    covered = []
    for off, n in blocks:
        covered.extend(range(off, off + n))
    assert covered == list(range(B))
    sizes = [n for _, n in blocks]
    assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    import oracle as O
    import workloads as W

    wl = W.make_workload(plant="boom", N=80, rank=24, hidden=(8,), B=10, T=6)
    goals = (wl.x0 + 0.3).astype(np.float32)
    mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
    return wl, goals, mdl


def _local_fn(mdl, wl):
    import oracle as O

    def fn(theta, x0, goals, T, seed, off, B_global):
        r = O.rollout(mdl, wl.sizes, "xg", theta, wl.Q, wl.sigma_r, x0, goals, T, seed, traj_offset=off,
                      B_global=B_global)
        return r["cost"], torch.from_numpy(r["grad"].astype(np.float64))

    return fn


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl, goals, mdl = _problem()
        cost, grad = rollout_cost_and_grad_dp(_local_fn(mdl, wl), wl.theta, wl.x0, goals, wl.T, 0x5EED0001)
        q.put((rank, cost, grad.numpy()))
    finally:
        tdist.destroy_process_group()


def test_two_rank_gloo_equals_single_process():
    import oracle as O

    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl, goals, mdl = _problem()
    ref = O.rollout(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.x0, goals, wl.T, 0x5EED0001)
    for rank, cost, grad in res:
        assert cost == pytest.approx(ref["cost"], rel=1e-13)
        assert np.allclose(grad, ref["grad"], rtol=1e-12, atol=1e-16)
    # both ranks hold bit-identical results after the all_reduce
    assert res[0][1] == res[1][1] and np.array_equal(res[0][2], res[1][2])


def test_allreduce_is_identity_without_process_group():
    g = torch.arange(5, dtype=torch.float32)
    c, g2 = allreduce_cost_grad(1.5, g)
    assert c == 1.5 and g2 is g
