# End-of-milestone check: build + smoke + full GPU tests + round profile
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/smoke.log
timeout 1500 bash scripts/gpu_tests.sh > /dev/null 2>&1
OUT=${OUT:-r01_e} bash scripts/prof_round.sh > /dev/null 2>&1
bash scripts/prof_list.sh > /dev/null 2>&1
echo done
