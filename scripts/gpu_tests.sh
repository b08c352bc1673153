cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -n "$K_EXPR" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rA -k "$K_EXPR" 2>&1 | tail -${TAIL:-60} > gpurun_out/gpu_tests.log
else
  timeout 1500 python -m pytest tests -m gpu -q -rA 2>&1 | tail -${TAIL:-60} > gpurun_out/gpu_tests.log
fi
echo done
