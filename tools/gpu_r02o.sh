#!/bin/bash
# r02o evidence: init early-exit A/B (config B launch lists), GPU tests, smoke, both bench arms at
# config C, the config-C launch list.
mkdir -p gpurun_out
for lp in -8 8; do
  SBO_INIT_LP=$lp timeout 300 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/initab_$lp.csv \
    python tools/profile_iteration.py --m 1048576 --scene 2048 > gpurun_out/initab_$lp.log 2>&1
  echo "== LP=$lp $(tail -2 gpurun_out/initab_$lp.log | head -1)"
  python tools/launch_summary.py gpurun_out/initab_$lp.csv | grep -E "init_block|polar_ns|total"
done
timeout 1500 python -m pytest tests -m gpu -q -rfs --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], d['phases_ms'], d['clocks'])"
tail -c 300 gpurun_out/bench_ref.log
timeout 900 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv python tools/profile_iteration.py > gpurun_out/launches.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 30 > gpurun_out/launch_summary.txt 2>&1; head -8 gpurun_out/launch_summary.txt
