# Round profile: full bench line, ncu launch list of a short bench, ncu --set full of the GP kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b_plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU:-k_p1_tc|k_p2_tc}" -s ${SKIP:-40} -c ${COUNT:-2} -o gpurun_out/${OUT:-prof} \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo done
