#!/bin/bash
# Quick loop: GPU parity tests, bench (no CPU baseline), launch list, optional ncu specs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
tail -c 2500 gpurun_out/bench.log
timeout 900 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_iteration.py > gpurun_out/launches.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 14
[ -n "$NCU_SPECS" ] && bash tools/gpu_prof.sh
exit 0
