# ncu --set full capture of the named kernels (regex in $NCU) on a short bench run
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python bench.py --config ${CONFIG:-C2} --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU" -s ${SKIP:-20} -c ${COUNT:-4} -o gpurun_out/${OUT:-prof} \
    python bench.py --config ${CONFIG:-C2} --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
