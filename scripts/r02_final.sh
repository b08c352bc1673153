# Round-end measurement set (one gpurun call): GPU suite, default bench line, its ncu launch list,
# the reference arm.  Outputs under gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/i_gpu_tests_full.log 2>&1
tail -40 gpurun_out/i_gpu_tests_full.log > gpurun_out/i_gpu_tests.log
timeout 900 python bench.py > gpurun_out/i_bench_c5.json 2> gpurun_out/i_bench_c5.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/i_c5_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/i_c5_ncu_stdout.txt 2>&1
python scripts/ncu_agg.py gpurun_out/i_c5_launches.csv > gpurun_out/i_c5_launch_summary.txt 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/i_ref_c5.json 2> gpurun_out/i_ref_c5.err
echo done
