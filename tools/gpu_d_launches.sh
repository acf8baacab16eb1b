#!/bin/bash
# Config D (p = 256, K = 32, s0 = 16) launch list of one iteration at m = 2^20.
mkdir -p gpurun_out
make -s -j8 > /dev/null 2>&1
timeout 900 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches_D.csv python tools/profile_iteration.py --m ${DM:-1048576} --scene 4096 --p-edge 16 --K 32 --s0 16 > gpurun_out/launches_D.log 2>&1
python tools/launch_summary.py gpurun_out/launches_D.csv 24
