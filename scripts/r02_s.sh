cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_train.py -q -rA -x -k "wide or c3 or maximum or train" > gpurun_out/r02s_tests.log 2>&1; echo "rc $?" >> gpurun_out/r02s_tests.log
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02s_c3.json 2>&1
