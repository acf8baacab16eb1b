#!/bin/bash
# Config D (p = 256, K = 32, s0 = 16) launch list at m = 2^20 and an ncu capture
# of the float64 re-decision.
mkdir -p gpurun_out
timeout 900 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_D.csv python tools/profile_iteration.py --m 1048576 --scene 4096 --p-edge 16 --K 32 --s0 16 > gpurun_out/launches_D.log 2>&1
python tools/launch_summary.py gpurun_out/launches_D.csv 20
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "iteration/" \
  -k regex:k_energy_f64 -s 1 -c 1 -o gpurun_out/full_recheckD -f python tools/profile_iteration.py --m 1048576 --scene 4096 --p-edge 16 --K 32 --s0 16 > gpurun_out/ncu_recheckD.log 2>&1
tail -1 gpurun_out/ncu_recheckD.log
