cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for f in 0 1; do
  BAGEL_P1_FUSED=$f timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$f.json 2> gpurun_out/ab_$f.err
done
BAGEL_P1_FUSED=1 timeout 120 python scripts/diag_timeline.py > gpurun_out/timeline.log 2>&1
