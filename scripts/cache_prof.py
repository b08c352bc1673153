"""Builds one workload's LOVE cache (timed by the library) -- run under an ncu launch list for the
per-kernel split.  python scripts/cache_prof.py C5"""
import sys

sys.path.insert(0, ".")
import workloads as W  # noqa: E402
from paper_2202_13638_b200 import bagel  # noqa: E402

wl = W.config(sys.argv[1] if len(sys.argv) > 1 else "C5")
ctx = bagel.Context(0)
ctx.gp_load(wl.X, wl.Y, wl.ell, wl.s, wl.noise)
print("cache build s", ctx.love_cache_build(wl.rank))
