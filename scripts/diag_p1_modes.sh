cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for m in ${MODES:-0 1 2 3}; do
  echo "== BAGEL_P1_DIAG=$m"
  BAGEL_P1_DIAG=$m timeout 120 python scripts/diag_timeline.py 2>&1 | head -8
done
