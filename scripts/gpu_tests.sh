cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -n "$K_EXPR" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rA -k "$K_EXPR" > gpurun_out/gpu_tests_full.log 2>&1
else
  timeout 1500 python -m pytest tests -m gpu -q -rA > gpurun_out/gpu_tests_full.log 2>&1
fi
tail -${TAIL:-60} gpurun_out/gpu_tests_full.log > gpurun_out/gpu_tests.log
echo done
