cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/diag_chain.py gpurun_out/r02f 80 9 6 3 > gpurun_out/r02f_chain.log 2>&1
