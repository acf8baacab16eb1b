#!/bin/bash
# A/B of library builds on one box: SBO_LIB=<name> python bench.py (short), alternating.
# usage: tools/ab.sh libA.so libB.so [extra bench args]
mkdir -p gpurun_out
A=$1; B=$2; shift 2
for rep in 1 2; do
  for L in $A $B; do
    SBO_LIB=$L timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/ab_$L.$rep.log 2>&1
    python - "$L" "$rep" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.{sys.argv[2]}.log").read().strip().splitlines()[-1])
    print(sys.argv[1], sys.argv[2], round(d["ms_per_step"], 3), {k: round(v, 2) for k, v in d["phases_ms"].items()})
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
  done
done
