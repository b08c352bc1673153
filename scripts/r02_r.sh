cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
P=gpurun_out/prof
timeout 300 python scripts/prof_kernels.py C2 100 > $P/r_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p1_tc|k_p2_tc" -s 20 -c 2 \
    -o $P/r_c2 python scripts/prof_kernels.py C2 100 > $P/r_ncu.log 2>&1
ncu -i $P/r_c2.ncu-rep --page source --csv --print-source sass > $P/r_c2_sass.csv 2>/dev/null
