#!/bin/bash
# r02r evidence at HEAD (cross terms first, certificate 3.3e-6): every GPU test, smoke, our bench arm, launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rfs --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], d['phases_ms'], d['clocks'])"
timeout 900 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv python tools/profile_iteration.py > gpurun_out/launches.log 2>&1
head -1 gpurun_out/launches.log
python tools/launch_summary.py gpurun_out/launches.csv 30 > gpurun_out/launch_summary.txt 2>&1; head -8 gpurun_out/launch_summary.txt
