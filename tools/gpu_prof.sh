#!/bin/bash
# Targeted ncu captures: NCU_SPECS="name:regex:skip ..." (one launch each) of tools/profile_iteration.py
mkdir -p gpurun_out
for spec in $NCU_SPECS; do
  IFS=: read name rx skip <<< "$spec"
  timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "iteration/" \
     -k regex:$rx -s $skip -c 1 -o gpurun_out/full_$name -f python tools/profile_iteration.py > gpurun_out/ncu_$name.log 2>&1
  tail -1 gpurun_out/ncu_$name.log
done
