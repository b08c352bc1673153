cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -rA -x --timeout=120 -k "both_gp_kernels or rank_above" 2>&1 | tail -60 > gpurun_out/gpu_tc.log
nvidia-smi --query-gpu=name,utilization.gpu --format=csv >> gpurun_out/gpu_tc.log
echo done
