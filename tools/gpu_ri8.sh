#!/bin/bash
# round_i8 check: parity tests, a short config-C bench, the launch list.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_round_i8.py -x -q -rf --timeout 100 > gpurun_out/pytest_ri8.log 2>&1
tail -15 gpurun_out/pytest_ri8.log
if grep -q " passed" gpurun_out/pytest_ri8.log && ! grep -q "failed\|error" gpurun_out/pytest_ri8.log; then
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_ri8.log 2>&1
  tail -c 400 gpurun_out/bench_ri8.log
  timeout 600 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/launches_ri8.csv python tools/profile_iteration.py > gpurun_out/launches_ri8.log 2>&1
  python tools/launch_summary.py gpurun_out/launches_ri8.csv 16
fi
mkdir -p gpurun_out
if grep -q " passed" gpurun_out/pytest_ri8.log; then timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "iteration/" \
  -k regex:k_round_i8 -s 7 -c 1 -o gpurun_out/full_ri8 -f python tools/profile_iteration.py --m 1048576 --scene 2048 > gpurun_out/ncu_ri8.log 2>&1; fi
tail -3 gpurun_out/ncu_ri8.log
