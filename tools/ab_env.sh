#!/bin/bash
# A/B of an environment switch on one box: tools/ab_env.sh VAR valueA valueB [bench args]
mkdir -p gpurun_out
V=$1; A=$2; B=$3; shift 3
for rep in 1 2; do
  for X in $A $B; do
    env $V=$X timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/abenv_$X.$rep.log 2>&1
    python - "$V" "$X" "$rep" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/abenv_{sys.argv[2]}.{sys.argv[3]}.log").read().strip().splitlines()[-1])
    print(sys.argv[1], sys.argv[2], sys.argv[3], round(d["ms_per_step"], 3), {k: round(v, 2) for k, v in d["phases_ms"].items()})
except Exception as e:
    print(sys.argv[2], "failed", e)
PY
  done
done
