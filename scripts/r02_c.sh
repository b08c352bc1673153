cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/diag_jv.py gpurun_out/r02c_jv.json > gpurun_out/r02c_jv.log 2>&1; echo "rc $?" >> gpurun_out/r02c_jv.log
bash scripts/r02_prof.sh > gpurun_out/r02c_prof.log 2>&1
