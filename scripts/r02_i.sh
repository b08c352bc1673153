cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/diag_comp.py gpurun_out/r02i > gpurun_out/r02i.log 2>&1
