cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python scripts/diag_fullbatch.py gpurun_out/r02d_fb 1 2 3 4 > gpurun_out/r02d_fb.log 2>&1
timeout 600 python scripts/diag_jv.py gpurun_out/r02d_jv.json > gpurun_out/r02d_jv.log 2>&1; echo "rc $?" >> gpurun_out/r02d_jv.log
