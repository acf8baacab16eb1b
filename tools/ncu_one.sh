#!/bin/bash
# ncu --set full of one retrain launch of kernel regex $1 (skip $2 launches) in tools/profile_iteration.py
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "iteration/" \
  -k regex:$1 -s ${2:-6} -c 1 -o gpurun_out/full_$3 -f python tools/profile_iteration.py > gpurun_out/ncu_$3.log 2>&1
tail -2 gpurun_out/ncu_$3.log
