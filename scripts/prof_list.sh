# ncu launch list (durations only) of the rollout kernels of a short bench run
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_p1_tc|k_p2_tc|k_r1a_tc|k_r1b_tc|k_init|k_reverse2|k_theta_grad|k_reduce|k_transpose_theta|k_epilogue" -c 5000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
echo done
