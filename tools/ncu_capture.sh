#!/bin/bash
# Full ncu captures (one launch each) of the iteration's top kernels.
set -x
mkdir -p gpurun_out
for k in k_polar k_energy_tc k_code_f64 k_outer_f64; do
  timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "iteration/" \
     -k regex:$k -c 1 -o gpurun_out/full_$k -f python tools/profile_iteration.py > gpurun_out/ncu_$k.log 2>&1
  tail -2 gpurun_out/ncu_$k.log
done
