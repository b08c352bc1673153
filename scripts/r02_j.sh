cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python scripts/diag_abs_v0.py gpurun_out/r02j > gpurun_out/r02j.log 2>&1
