#!/bin/bash
# Round-2 evidence: shim tests (baseline/_ref), the sharded bench on one GPU, the
# config-C launch list, ncu --set full captures of the top kernels and of the
# HBM-bound select / group / sum passes.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_orthodict_shim.py -q -rs > gpurun_out/pytest_shim.log 2>&1; tail -2 gpurun_out/pytest_shim.log
SBO_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --m-total 1048576 --no-cpu-baseline --no-e2e > gpurun_out/bench_2r.log 2>&1
tail -c 400 gpurun_out/bench_2r.log; echo
timeout 900 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv python tools/profile_iteration.py > gpurun_out/launches.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 30 > gpurun_out/launch_summary.txt 2>&1; head -12 gpurun_out/launch_summary.txt
for spec in ${NCU_SPECS:-"round_i8:k_round_i8:7 energy16:k_energy_tc:1 outer_i8:k_outer_i8:7 key_hist:k_key_hist:0 group_scatter:k_group_scatter:1 sum_tiles:k_sum_tiles:0 y_tiles:k_y_tiles:1"}; do
  IFS=: read name rx skip <<< "$spec"
  timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "iteration/" \
     -k regex:$rx -s $skip -c 1 -o gpurun_out/full_$name -f python tools/profile_iteration.py > gpurun_out/ncu_$name.log 2>&1
  tail -1 gpurun_out/ncu_$name.log
done
