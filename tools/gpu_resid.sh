#!/bin/bash
# ncu --set full of the residual-mode k_round_i8 launch (represent #2) and of a code-mode launch at config C
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "iteration/" \
  -k regex:k_round_i8 -s 12 -c 1 -o gpurun_out/full_ri8_resid -f python tools/profile_iteration.py > gpurun_out/ncu_ri8_resid.log 2>&1
tail -2 gpurun_out/ncu_ri8_resid.log
