# C5 --set full of the GP-step kernels (step 1 of a T = 3 rollout) + dram bytes of every kernel at C2/C3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
P=gpurun_out/prof
timeout 300 python scripts/prof_kernels.py C5 3 > $P/c5_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p1_tc|k_p2_tc|k_r1a_tc|k_r1b_tc" -s 5 -c 4 \
    -o $P/c5_full python scripts/prof_kernels.py C5 3 > $P/c5_ncu.log 2>&1
timeout 300 python scripts/prof_kernels.py C2 100 2 > $P/c2_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 3000 --csv \
    --log-file $P/c2_list.csv python scripts/prof_kernels.py C2 100 2 > $P/c2_ncu.log 2>&1
timeout 300 python scripts/prof_kernels.py C3 20 > $P/c3_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 3000 --csv \
    --log-file $P/c3_list.csv python scripts/prof_kernels.py C3 20 > $P/c3_ncu.log 2>&1
ls -la $P
