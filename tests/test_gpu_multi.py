"""Multi-GPU data parallelism on real GPUs: torchrun with 2 ranks over NCCL -- sharded
rollout + one all_reduce equals the single-GPU full batch (relative 1e-6; the per-trajectory
arithmetic is bit-identical, only the theta-gradient summation order differs), the replicated LOVE
caches are bit-identical across ranks, and a repeated iteration is bitwise equal (NCCL algorithm and
protocol pinned).  Skipped when fewer than 2 GPUs are visible (the pool's boxes have one; the host
logic is covered on CPU by tests/test_dist_gloo.py)."""
import json
import os
import subprocess
import sys

import pytest
import torch

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_two_rank_nccl_equals_single_gpu():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "scripts", "dp_check.py"), "C2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-2000:] + r.stderr[-2000:]
    out = json.loads(lines[-1])
    assert out["ok"], out
