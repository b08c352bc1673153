"""tcgen05.mma issue-rate microbenchmark (GPU box): cycles per MMA for M=128, K=16 vs N,
loop unrolling and independent accumulators."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2202_13638_b200 import bagel  # noqa: E402

ctx = bagel.Context(0)
for ts in (0, 1):
    for N in (32, 64, 128, 256):
        for nacc in (1, 2):
            if nacc * N > 256:
                continue
            mode = ts | (nacc << 1) | 16
            ctx.tc_bench(N, 64, mode, 148)
            cyc = ctx.tc_bench(N, 4096, mode, 148)
            per = cyc.mean() / 4096
            ideal = 128 * N / 256
            print(f"unrolled {'TS' if ts else 'SS'} N={N:3d} nacc={nacc}: {per:7.1f} cycles/MMA "
                  f"(ideal {ideal:5.1f}, {ideal / per:5.1%} of peak)", flush=True)
