cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rA -x > gpurun_out/r02a_tests.log 2>&1; echo "tests rc $?" >> gpurun_out/r02a_tests.log
timeout 900 python bench.py --config C5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02a_bench_c5.log 2>&1; echo "rc $?" >> gpurun_out/r02a_bench_c5.log
