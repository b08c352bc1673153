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


class _OracleCtx:
    """Stand-in for bagel.Context on CPU (test-only): the oracle's sampler, rollout and Adam behind the
    methods train.train_policy calls, so the loop's sharding and all_reduce are exercised without a GPU."""

    def __init__(self, mdl, wl):
        self.mdl, self.wl = mdl, wl
        self.dev = torch.device("cpu")

    def sample_states(self, seed, off, B, lo, hi, which=0, out=None):
        import oracle as O

        out.copy_(torch.from_numpy(O.sample_states(seed, off, B, lo, hi, which).astype(np.float32)))
        return out

    def rollout_cost_and_grad(self, theta, x0, goals, T, seed, traj_offset=0, B_global=None, grad=None):
        import oracle as O

        r = O.rollout(self.mdl, self.wl.sizes, "xg", theta.double().numpy(), self.wl.Q, self.wl.sigma_r,
                      x0.double().numpy(), goals.double().numpy(), T, seed, traj_offset=traj_offset,
                      B_global=B_global)
        grad.copy_(torch.from_numpy(r["grad"]))
        return r["cost"], grad

    def adam_step(self, params, grad, m1, m2, step, lr=1e-2, beta1=0.9, beta2=0.999, eps=1e-8, report_skip=False):
        import oracle as O

        th, g = params.double().numpy().copy(), grad.double().numpy().copy()
        a, b = m1.double().numpy().copy(), m2.double().numpy().copy()
        skipped = O.adam_step(th, g, a, b, step, lr, beta1, beta2, eps)
        params.copy_(torch.from_numpy(th))
        m1.copy_(torch.from_numpy(a))
        m2.copy_(torch.from_numpy(b))
        return skipped


def _train_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_13638_b200.train import train_policy

        wl, _, mdl = _problem()
        lo, hi = wl.X[:, :wl.p].min(0), wl.X[:, :wl.p].max(0)
        th, log = train_policy(_OracleCtx(mdl, wl), wl.theta, wl.T, 4, wl.B, lo, hi, lr=1e-2, seed0=0x5EED2000)
        q.put((rank, log.cost, th.double().numpy()))
    finally:
        tdist.destroy_process_group()


def test_two_rank_training_loop_equals_single_process():
    """Algorithm 1's loop (train.train_policy) at world size 2: each rank samples and rolls out its own
    trajectory block, one all_reduce per iteration, identical replicated Adam updates -- equal to the
    single-process oracle loop (O.train) on the whole batch."""
    import oracle as O

    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_train_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl, _, mdl = _problem()
    lo, hi = wl.X[:, :wl.p].min(0), wl.X[:, :wl.p].max(0)
    th_ref, costs_ref = O.train(mdl, wl.sizes, "xg", wl.theta, wl.Q, wl.sigma_r, wl.T, 4, wl.B, lo, hi, 0x5EED2000,
                                lr=1e-2)
    (_, c0, t0), (_, c1, t1) = sorted(res, key=lambda r: r[0])
    assert np.array_equal(t0, t1)  # replicated parameters stay identical on every rank
    np.testing.assert_allclose(c0, costs_ref, rtol=1e-5)
    np.testing.assert_allclose(t0, th_ref, rtol=1e-5, atol=1e-6)


class _CacheCtx:
    """Stand-in exposing cache_get (alpha, R per output) on CPU for the replicated-cache check."""

    def __init__(self, rank, corrupt):
        self.dev = torch.device("cpu")
        g = torch.Generator().manual_seed(5)
        self.a = [torch.randn(50, generator=g, dtype=torch.float64) for _ in range(2)]
        self.R = [torch.randn(7, 50, generator=g, dtype=torch.float64) for _ in range(2)]
        if corrupt and rank == 1:
            self.R[1][3, 17] = torch.nextafter(self.R[1][3, 17], torch.tensor(1e9, dtype=torch.float64))

    def cache_get(self, m):
        return self.a[m], self.R[m]


def _cache_worker(rank, world, port, corrupt, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2202_13638_b200.dist import verify_replicated_cache

        try:
            verify_replicated_cache(_CacheCtx(rank, corrupt), 2)
            q.put((rank, "same"))
        except RuntimeError:
            q.put((rank, "differ"))
    finally:
        tdist.destroy_process_group()


@pytest.mark.parametrize("corrupt", [False, True])
def test_replicated_cache_check_detects_one_ulp(corrupt):
    """the LOVE cache is replicated, each rank building it deterministically; the bench
    checks the copies are bit-identical across ranks -- one ulp of one R entry on one rank is caught."""
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_cache_worker, args=(r, world, port, corrupt, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert {r[1] for r in res} == {"differ" if corrupt else "same"}


def test_nccl_algorithm_and_protocol_are_pinned(monkeypatch):
    from paper_2202_13638_b200.dist import pin_nccl

    monkeypatch.delenv("NCCL_ALGO", raising=False)
    monkeypatch.delenv("NCCL_PROTO", raising=False)
    pin_nccl()
    assert os.environ["NCCL_ALGO"] == "Ring" and os.environ["NCCL_PROTO"] == "LL"


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_strong_scaling_shards_c5_batch(world):
    """bench.py's default strong scaling: C5's 65,536 trajectories split over the launched world,
    contiguous global ids, every trajectory exactly once (8,192 per GPU at 8 GPUs)."""
    blocks = [shard(65536, world, r) for r in range(world)]
    assert sum(n for _, n in blocks) == 65536
    assert all(n == 65536 // world for _, n in blocks)
    assert [o for o, _ in blocks] == [r * (65536 // world) for r in range(world)]
