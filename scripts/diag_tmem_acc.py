"""Diagnostic (GPU box): rounding of tcgen05 fp32 accumulation in TMEM.  One CTA accumulates
D = A . B^T over K = 16 * steps with positive fp16 operands (partial sums grow, so a truncating
accumulator shows a bias that grows linearly with the chain length; round-to-nearest shows a
sqrt-like random walk).  Printed: mean and max of (D - exact) / (steps * ulp(D)) and the fraction of
entries below the exact value, against the same chain summed in fp32 round-to-nearest on the CPU."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_13638_b200 import bagel  # noqa: E402



def pack(M):
    """Canonical no-swizzle K-major packing (csrc/tc.cuh canon_idx) of an R x K fp16 matrix."""
    R, K = M.shape
    out = np.empty(R * K, dtype=np.float16)
    r = np.arange(R)[:, None]
    k = np.arange(K)[None, :]
    idx = (((r >> 3) * (K >> 3) + (k >> 3)) << 6) + ((r & 7) << 3) + (k & 7)
    out[idx.reshape(-1)] = M.reshape(-1)
    return out


ctx = bagel.Context(0)
rng = np.random.default_rng(0)
N = 16


def run(A, B):
    K = A.shape[1]
    a = torch.from_numpy(pack(A).view(np.int16)).cuda()
    b = torch.from_numpy(pack(B).view(np.int16)).cuda()
    return ctx.tc_selftest(a, b, N, K, 0).cpu().numpy().astype(np.float64)


for kind in ("positive", "signed", "positive+offset"):
    for K in (16, 64, 256, 672):
        A = rng.uniform(0.5, 1.0, (128, K)).astype(np.float16)
        B = rng.uniform(0.5, 1.0, (N, K)).astype(np.float16)
        if kind == "signed":
            B = (B * rng.choice([-1.0, 1.0], (N, K))).astype(np.float16)
        ex = A.astype(np.float64) @ B.astype(np.float64).T
        if kind.endswith("offset"):
            # first K block adds C = 16 * 1 * 2^10 = 2^14 exactly: every partial sum then has the exponent of C
            A2 = np.concatenate([np.ones((128, 16), np.float16), A], 1)
            B2 = np.concatenate([np.full((N, 16), 1024.0, np.float16), B], 1)
            D = run(A2, B2) - 16384.0
            ulp = np.full_like(ex, np.spacing(np.float32(16384.0 + ex.max())), dtype=np.float64)
        else:
            D = run(A, B)
            ulp = np.spacing(np.abs(ex).astype(np.float32)).astype(np.float64)
        rn = np.zeros_like(ex, dtype=np.float32)
        for st in range(K // 16):
            blk = A[:, 16 * st:16 * st + 16].astype(np.float64) @ B[:, 16 * st:16 * st + 16].astype(np.float64).T
            rn = (rn.astype(np.float64) + blk).astype(np.float32)
        e = (D - ex) / ulp
        r = (rn.astype(np.float64) - ex) / np.spacing(np.abs(ex).astype(np.float32)).astype(np.float64)
        print(f"{kind:16s} K={K:4d} steps={K // 16:3d}: tensor core err/ulp mean {e.mean():+.3f} std {e.std():.3f} "
              f"max|.| {np.abs(e).max():.2f} frac<exact {np.mean(D < ex):.2f} | fp32 RN chain mean {r.mean():+.3f} "
              f"max|.| {np.abs(r).max():.2f}", flush=True)
