cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/r02h_tests.log 2>&1; echo "rc $?" >> gpurun_out/r02h_tests.log
timeout 600 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_bench_c2.log 2>&1
