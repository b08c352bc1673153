cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_tc.py -q -rA > gpurun_out/r02l_tc.log 2>&1
