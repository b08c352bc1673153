cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
P=gpurun_out/prof
timeout 300 python scripts/prof_kernels.py C5 3 > $P/c5o_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p2_tc" -s 1 -c 1 \
    -o $P/c5_p2 python scripts/prof_kernels.py C5 3 > $P/c5o_ncu.log 2>&1
ncu -i $P/c5_p2.ncu-rep --page source --csv --print-source sass > $P/c5_p2_sass.csv 2>/dev/null
ls -la $P
