cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
DIAG_NO_PERTURB=1 timeout 900 python scripts/diag_c2_grad.py gpurun_out/r02g_grad.json 3 > gpurun_out/r02g_diag.log 2>&1
