cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/diag_tmem_acc.py > gpurun_out/r02e_tmem.log 2>&1
