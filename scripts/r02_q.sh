cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/prof
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r02q_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/r02q_smoke.log
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/r02q_tests.log 2>&1; echo "rc $?" >> gpurun_out/r02q_tests.log
timeout 1200 python bench.py > gpurun_out/r02q_bench_c5.json 2> gpurun_out/r02q_bench_c5.err
P=gpurun_out/prof
timeout 300 python scripts/prof_kernels.py C5 3 > $P/q_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_p1_tc|k_p2_tc|k_r1a_tc|k_r1b_tc|k_epilogue|k_reverse2|k_theta_grad" -s 5 -c 7 \
    -o $P/q_c5 python scripts/prof_kernels.py C5 3 > $P/q_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_p1_tc|k_p2_tc|k_r1a_tc|k_r1b_tc|k_epilogue|k_init|k_reverse2|k_theta_grad|k_reduce|k_transpose|k_mlp" -c 2000 --csv \
    --log-file $P/q_c2_list.csv python scripts/prof_kernels.py C2 100 2 > $P/q_c2_ncu.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_p1_tc|k_p2_tc|k_r1a_tc|k_r1b_tc|k_epilogue|k_init|k_reverse2|k_theta_grad|k_reduce|k_transpose|k_mlp" -c 2000 --csv \
    --log-file $P/q_c3_list.csv python scripts/prof_kernels.py C3 20 > $P/q_c3_ncu.log 2>&1
