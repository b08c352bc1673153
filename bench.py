#!/usr/bin/env python
"""BAGEL hot-path benchmark (BASELINE.json metric: trajectory-steps/sec (fwd+bwd) and
policy-grad iters/sec at 1/2/4/8 B200).

One "step" = one policy-gradient iteration = rollout_cost_and_grad over the rank's
trajectories (forward T steps through the LOVE-GP model + reverse pass) plus the single
gradient all_reduce when N > 1.  Default workload: BASELINE.json configs[4], the config the
metric is quoted on ("C5": GP N=50,000 on the boom plant's (pos, vel, valve cmd), LOVE rank
512, policy MLP 4-64-64-1, B=65,536 trajectories sharded over the GPUs, T=200), synthetic
boom-plant data (workloads/); strong scaling by default (B is the global batch).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--scaling strong|weak]
                    [--impl reference]

Prints ONE JSON line on rank 0.  Timing: CUDA events on the context stream around each
timed iteration, L2 flushed (256 MiB write) between iterations outside the events,
barrier + synchronize on both sides of the timed region, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "trajectory-steps/sec (fwd+bwd)"
UNIT = "traj-steps/s"


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """SM clocks / throttle reasons sampled DURING the timed region: NVML every ~2 ms from a thread
    (the timed region of the default run is only ~0.1 s), nvidia-smi -lms 100 if NVML is missing."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.sm, self.reasons, self.mx = [], set(), None
        self.proc = self.nv = None
        self.stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as nv

            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                    "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                    "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                    "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            self.nv = nv

            def loop():
                while not self.stop.is_set():
                    try:
                        self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        self.reasons.update(n for n, b in bits.items() if r & b)
                    except nv.NVMLError:
                        pass
                    time.sleep(0.002)

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            r = [c.strip() for c in line.split(",")]
            try:
                self.sm.append(float(r[1]))
                self.mx = float(r[2])
                self.reasons.update(n for n, v in zip(self.NAMES, r[5:9]) if v.lower().startswith("active"))
            except (ValueError, IndexError):
                continue

    def __exit__(self, *a):
        self.stop.set()
        if self.nv is not None:
            self.thread.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        return {"sm_mhz": float(np.median(self.sm)) if self.sm else None, "sm_max_mhz": self.mx,
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml" if self.nv is not None else "nvidia-smi"}


def flops_per_traj_step(wl):
    """Algorithmic tensor-eligible flops of the GP contraction:
    pass 1 (a3): 2 p N (1 + d + k); pass 2 (a5): 2 p N k + 2 p N (1 + d)."""
    p, N, d, k = wl.p, wl.N, wl.d, wl.rank
    return 2 * p * N * (1 + d + k), 2 * p * N * k + 2 * p * N * (1 + d)


# largest N whose oracle cache (fp64 Cholesky for alpha + the naive dense LOVE build) the oracle
# builds itself within the bench's few-minute budget; above it the oracle takes the GPU-built alpha
# and R (permitted at C5, declared in the sample string)
ORACLE_OWN_CACHE_MAX_N = 20000


def oracle_model(wl, ctx=None):
    """(oracle Model, how its cache was made).  ctx: a bagel Context whose GPU-built cache may be
    imported when N is beyond ORACLE_OWN_CACHE_MAX_N (cpu_baseline leg only)."""
    import oracle as O

    if wl.N <= ORACLE_OWN_CACHE_MAX_N:
        t0 = time.perf_counter()
        mdl = O.Model.build(wl.X, wl.Y, wl.ell, wl.s, wl.noise, wl.rank)
        return mdl, f"oracle's own cache build {time.perf_counter() - t0:.1f} s (excluded)"
    if ctx is None:
        return None, None
    al, Rs = [], []
    for m in range(wl.p):
        a, R = ctx.cache_get(m)
        al.append(a.cpu().numpy())
        Rs.append(R.cpu().numpy())
    return (O.Model(wl.X, wl.ell, wl.s, np.stack(al), np.stack(Rs)),
            "alpha and R built on the GPU and imported into the oracle (N > %d, SURVEY §8(d))" % ORACLE_OWN_CACHE_MAX_N)


def cpu_baseline(wl, ctx=None, budget_s=20.0, max_traj=256):
    """Oracle (float64 C, OpenMP over trajectories) on a bounded trajectory subset, full N, k, T."""
    import oracle as O

    cores = len(os.sched_getaffinity(0))
    O.set_num_threads(cores)
    mdl, how = oracle_model(wl, ctx)
    phi = "xg" if wl.sizes[0] == 2 * wl.p else "xgd"
    n, total_t, total_steps = 4, 0.0, 0
    while True:
        n = min(n, max_traj, wl.B)
        t0 = time.perf_counter()
        O.rollout(mdl, wl.sizes, phi, wl.theta, wl.Q, wl.sigma_r, wl.x0[:n], wl.goals[:n], wl.T,
                  W.rollout_seed(0), B_global=wl.B)
        dt = time.perf_counter() - t0
        total_t += dt
        total_steps += n * wl.T
        if total_t + 2.2 * dt >= budget_s or n >= max_traj or n >= wl.B:
            break
        n *= 2
    return {"value": total_steps / total_t, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{total_steps // wl.T} trajectories x T={wl.T} (full N={wl.N}, k={wl.rank}) fwd+bwd in "
                      f"{total_t:.1f} s; {how}"}


def run_reference(args, wl, rank, world):
    """--impl reference: the oracle as it stands on the host cores (this tier's reference arm), on a
    bounded per-step sample of the same workload.  Never loads libbagel.so."""
    if rank != 0:
        return
    import oracle as O

    cores = len(os.sched_getaffinity(0))
    O.set_num_threads(cores)
    base = {"impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": config_dict(args, wl, world)}
    mdl, how = oracle_model(wl)
    if mdl is None:
        # the oracle's own exact-alpha Cholesky (N^3/3 = 4e13 flops at N = 50,000) and dense LOVE
        # build (20 GB K-hat) take tens of minutes on the host; this arm may not borrow the GPU's cache
        line = dict(base, value=None, ms_per_step=None,
                    reason=f"the oracle cannot build its own LOVE cache at N={wl.N} within the bench budget "
                           f"(exact Cholesky ~{wl.N ** 3 / 3:.1e} flop per output); the same oracle timed "
                           f"with the GPU-built cache is this run's cpu_baseline in the default arm",
                    cpu_baseline={"value": None, "unit": UNIT, "cores": cores, "kind": "oracle",
                                  "sample": "none (cache not buildable by the oracle in time)"},
                    e2e={"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
        print(json.dumps(line), flush=True)
        return
    phi = "xg" if wl.sizes[0] == 2 * wl.p else "xgd"
    # per-step sample: about 20 s of oracle work per step at most, whole run within a few minutes
    t0 = time.perf_counter()
    O.rollout(mdl, wl.sizes, phi, wl.theta, wl.Q, wl.sigma_r, wl.x0[:1], wl.goals[:1], wl.T,
              W.rollout_seed(0), B_global=wl.B)
    per_traj = time.perf_counter() - t0
    budget = 180.0 / max(1, args.steps + args.warmup)
    n = int(max(1, min(wl.B, args.ref_traj or 10 ** 9, budget / max(per_traj, 1e-6) * min(cores, 8))))
    for i in range(args.warmup):
        O.rollout(mdl, wl.sizes, phi, wl.theta, wl.Q, wl.sigma_r, wl.x0[:n], wl.goals[:n], wl.T,
                  W.rollout_seed(i), B_global=wl.B)
    times = []
    for i in range(args.steps):
        t0 = time.perf_counter()
        O.rollout(mdl, wl.sizes, phi, wl.theta, wl.Q, wl.sigma_r, wl.x0[:n], wl.goals[:n], wl.T,
                  W.rollout_seed(args.warmup + i), B_global=wl.B)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = n * wl.T * args.steps / tot
    line = dict(base, value=value, ms_per_step=1e3 * tot / args.steps,
                cpu_baseline={"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                              "sample": f"{n} of {wl.B} trajectories per step, full N={wl.N}, k={wl.rank}, "
                                        f"T={wl.T}; {how}"},
                e2e={"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0})
    print(json.dumps(line), flush=True)


def config_dict(args, wl, world):
    per = "per GPU" if args.scaling == "weak" else "in total, sharded over the ranks"
    B_global = wl.B * world if args.scaling == "weak" else wl.B
    return {"workload": f"{args.config}: GP N={wl.N} d={wl.d} p={wl.p}, LOVE rank {wl.rank}, "
                        f"MLP {'-'.join(map(str, wl.sizes))}, B={wl.B} {per}, T={wl.T}",
            "global_batch": B_global, "horizon": wl.T, "parallelism": f"dp{world}",
            "l2": "flushed (256 MiB write) between timed iterations"}


def load_traffic(config, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` at `config`, from the
    committed ncu --set full capture (profiles/traffic.json); None if that capture does not exist."""
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(tpath) as f:
            return json.load(f).get(config, {}).get(kernel)
    except (OSError, ValueError):
        return None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    # BASELINE.json's metric is quoted on configs[4] ("C5: N=50,000, B=65,536 trajectories sharded over
    # 1/2/4/8 B200"): the default workload, strong scaling (B is the global batch)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--impl", default="bagel", choices=["bagel", "reference"])
    ap.add_argument("--ref-traj", type=int, default=0, help="reference arm: trajectories per step (0 = auto)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))  # the launched process group, never --gpus
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; reporting the launched world "
              f"({world}); launch N > 1 with torchrun", file=sys.stderr)
    wl = W.config(args.config)

    if args.impl == "reference":
        run_reference(args, wl, rank, world)
        return

    import torch
    import torch.distributed as tdist

    from paper_2202_13638_b200 import bagel
    from paper_2202_13638_b200.dist import allreduce_cost_grad, pin_nccl, shard, verify_replicated_cache

    torch.cuda.set_device(local)
    if world > 1:
        pin_nccl()
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    # strong scaling (default): the config's B trajectories split into contiguous per-rank blocks;
    # weak: B per GPU.  Global trajectory ids are contiguous per rank either way (eps by global id).
    B_global = wl.B if args.scaling == "strong" else wl.B * world
    x0g, gg = W.sample_states_goals(wl.X, wl.p, B_global)
    off, bl = shard(B_global, world, rank)

    ctx = bagel.setup(wl, device=local)
    cache_s = ctx.cache_seconds
    if world > 1:
        verify_replicated_cache(ctx, wl.p)   # every rank's LOVE cache bit-identical (deterministic build)
    theta = torch.from_numpy(wl.theta).to(dev)
    x0 = torch.from_numpy(x0g[off:off + bl]).to(dev)
    goals = torch.from_numpy(gg[off:off + bl]).to(dev)
    grad = torch.empty(ctx.n_params, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)

    def iteration(i):
        cost, g = ctx.rollout_cost_and_grad(theta, x0, goals, wl.T, W.rollout_seed(i), traj_offset=off,
                                            B_global=B_global, grad=grad)
        return allreduce_cost_grad(cost, g)

    w0 = time.perf_counter()
    for i in range(args.warmup):
        iteration(i)
    torch.cuda.synchronize()
    warm_ms = 1e3 * (time.perf_counter() - w0) / args.warmup
    # per-kernel CUDA events (roofline numerator): inside the timed region when a step is long
    # enough that ~4 event records per rollout step are noise (C4/C5: 2 launches of ~10-20 ms each per
    # step); otherwise in a separate pass of the same steps (C2: they would perturb a 5 ms step)
    inline_prof = warm_ms >= 500.0

    # ---------------- timed region (device-resident inputs)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    launches = 0
    if inline_prof:
        ctx.profile(True)
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))
            ev[i][0].record(stream)
            iteration(args.warmup + i)
            ev[i][1].record(stream)
            launches += ctx.last_launch_count()
        torch.cuda.synchronize()
    if world > 1:
        tdist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    if inline_prof:
        prof = ctx.profile_get()
        ctx.profile(False)
        prof_steps = args.steps
        prof_ms_per_step = None
    else:
        torch.cuda.synchronize()
        ctx.profile(True)
        prof_steps = args.steps
        pe0, pe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        pe0.record(stream)
        for i in range(prof_steps):
            flush.fill_(float(i))
            iteration(args.warmup + i)
        pe1.record(stream)
        torch.cuda.synchronize()
        prof = ctx.profile_get()
        ctx.profile(False)
        prof_ms_per_step = pe0.elapsed_time(pe1) / prof_steps
    tot_ms = float(sum(step_ms))
    t = torch.tensor([tot_ms], dtype=torch.float64, device=dev)
    if world > 1:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    tot_ms = float(t.item())
    ms_per_step = tot_ms / args.steps
    value = B_global * wl.T * args.steps / (tot_ms / 1e3)

    # ---------------- end-to-end: host (pinned) buffers through the C ABI, copies inside the timing
    th_h = torch.from_numpy(wl.theta).pin_memory()
    x0_h = torch.from_numpy(x0g[off:off + bl]).pin_memory()
    g_h = torch.from_numpy(gg[off:off + bl]).pin_memory()
    grad_h = torch.empty(ctx.n_params).pin_memory()
    e2e_steps = max(3, min(args.steps, 10 if ms_per_step < 1000 else 3))
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(e2e_steps):
        cost, g = ctx.rollout_cost_and_grad(th_h, x0_h, g_h, wl.T, W.rollout_seed(1000 + i), traj_offset=off,
                                            B_global=B_global, grad=grad if world > 1 else grad_h)
        if world > 1:
            cost, g = allreduce_cost_grad(cost, g)
            grad_h.copy_(g, non_blocking=True)
            stream.synchronize()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        tdist.all_reduce(e2e_ms, op=tdist.ReduceOp.MAX)
    e2e_value = B_global * wl.T * e2e_steps / (float(e2e_ms.item()) / 1e3)
    h2d = (ctx.n_params + 2 * bl * wl.p) * 4
    d2h = ctx.n_params * 4 + 8

    if rank == 0:
        pk, pk_kind = peaks()
        f1, f2 = flops_per_traj_step(wl)
        names = {"gp_pass1": f1, "gp_pass2": f2}
        dom = max(names, key=lambda n: prof[n][0])
        dom_ms, dom_n = prof[dom]
        per_launch_s = dom_ms / 1e3 / dom_n
        flops_launch = names[dom] * bl
        achieved = flops_launch / per_launch_s / 1e12
        # burst peak for a kernel inside a short step, sustained inside a seconds-long one
        sustained = ms_per_step >= 100.0
        peak = pk.get("bf16_tflops_sustained" if sustained else "bf16_tflops", 1363.2)
        traffic = load_traffic(args.config, dom)
        step_share = {k: round(v[0] / max(1e-9, sum(x[0] for x in prof.values())), 4) for k, v in prof.items()}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (boom-plant transitions, workloads/)",
            "config": config_dict(args, wl, world),
            "policy_grad_iters_per_s": 1e3 / ms_per_step,
            "step_ms_p10_p50_p90": [float(np.percentile(step_ms, q)) for q in (10, 50, 90)],
            "cache_build_s": cache_s,
            "roofline": {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": f"{pk_kind} bf16_tflops{'_sustained' if sustained else ''} "
                                        f"(fp16 kind::f16 runs at the bf16 rate; "
                                        f"{'sustained: seconds-long step' if sustained else 'burst: short step'})",
                         "traffic_source": "profiles/traffic.json (ncu --set full, dram read+write per launch)",
                         "algorithmic_flops_per_launch": flops_launch,
                         "issued_flops_per_launch": 3 * flops_launch,
                         "note": "3-pass fp16 hi/lo split: the tensor pipe issues 3x the algorithmic flops, "
                                 "so frac <= 1/3 by construction"},
            "kernel_ms_per_step": {k: v[0] / prof_steps for k, v in prof.items()},
            "kernel_share": step_share,
            "kernel_events": "inside the timed region" if inline_prof else
                             f"separate pass of {prof_steps} steps ({prof_ms_per_step:.3f} ms/step with events)",
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(wl, ctx)
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        tdist.destroy_process_group()


if __name__ == "__main__":
    main()
