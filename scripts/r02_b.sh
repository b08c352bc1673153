cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rA -x > gpurun_out/r02b_parity.log 2>&1; echo "rc $?" >> gpurun_out/r02b_parity.log
timeout 1500 python scripts/diag_c2_grad.py gpurun_out/r02b_grad.json 1 2 > gpurun_out/r02b_diag.log 2>&1; echo "rc $?" >> gpurun_out/r02b_diag.log
