#!/bin/bash
# Round-2 evidence session: parity tests, smoke, bench (both arms, config C default),
# ncu launch list of one config-C iteration.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt
timeout 1200 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv python tools/profile_iteration.py > gpurun_out/launches.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 30 > gpurun_out/launch_summary.txt 2>&1
tail -5 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log; tail -c 600 gpurun_out/bench.log; tail -c 600 gpurun_out/bench_ref.log; cat gpurun_out/launch_summary.txt
