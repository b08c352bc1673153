# usage: ENVS="A=0 A=1" bash scripts/ab_env.sh  -- one short bench per env setting
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
i=0
for e in $ENVS; do
  env ${e//+/ } timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$i.json 2> gpurun_out/ab_$i.err
  python - "$e" gpurun_out/ab_$i.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"] / 1e6, 3), "M", round(d["ms_per_step"], 3), "ms", {k: round(v, 3) for k, v in d["kernel_ms_per_step"].items()})
except Exception as ex:
    print(sys.argv[1], "FAILED", ex)
PY
  i=$((i+1))
done
