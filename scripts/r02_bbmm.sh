set -x
python scripts/bbmm_prof.py C4 8 100 2 && python scripts/bbmm_prof.py C4 16 100 1 && python scripts/bbmm_prof.py C5 8 100 1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv --log-file gpurun_out/bbmm_launches.csv python scripts/bbmm_prof.py C4 8 20 1 > /dev/null 2>&1
python scripts/ncu_agg.py gpurun_out/bbmm_launches.csv
timeout 900 python -m pytest tests/test_gpu_bbmm.py -q -x 2>&1 | tail -3
