cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tc.py tests/test_gpu_variants.py -q -rA -x > gpurun_out/r02p_tests.log 2>&1; echo "rc $?" >> gpurun_out/r02p_tests.log
timeout 300 python bench.py --config C2 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02p_c2.json 2>&1
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02p_c3.json 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02p_c5.json 2>&1
