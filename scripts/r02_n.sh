cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python - > gpurun_out/r02n_bench.log 2>&1 <<'PY'
import numpy as np
from paper_2202_13638_b200 import bagel
c = bagel.Context(0)
for N in (64, 128, 256):
    for mode, ctas, lab in ((0, 148, "SS 1cta"), (1, 148, "TS 1cta"), (64, 74, "SS pair M=256"), (65, 74, "TS pair M=256")):
        cyc = c.tc_bench(N, 4096, mode, ctas)
        print(f"N={N:3d} {lab:14s}: {np.median(cyc) / 4096:.1f} cycles per MMA (per {'pair' if mode >= 64 else 'SM'})", flush=True)
PY
