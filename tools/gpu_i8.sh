#!/bin/bash
# quick loop for the tensor-core outer product: its tests, then a short bench breakdown
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_outer_i8.py -q -rf -x --timeout 120 > gpurun_out/pytest_i8.log 2>&1
tail -3 gpurun_out/pytest_i8.log
timeout 600 python bench.py --steps 5 --no-cpu-baseline --no-e2e "$@" > gpurun_out/bench.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench.log").read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["phases_ms"])
for k, v in d["kernels"].items():
    print(k, v["launches"], round(v["ms_per_step"], 3))
PY
