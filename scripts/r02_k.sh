cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rA > gpurun_out/r02k_tests.log 2>&1; echo "rc $?" >> gpurun_out/r02k_tests.log
timeout 1200 python bench.py > gpurun_out/r02k_bench_c5.json 2> gpurun_out/r02k_bench_c5.err; echo "rc $?" >> gpurun_out/r02k_bench_c5.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02k_ref_c5.json 2>&1
timeout 900 python bench.py --config C2 --impl reference --steps 3 --warmup 1 > gpurun_out/r02k_ref_c2.json 2>&1
