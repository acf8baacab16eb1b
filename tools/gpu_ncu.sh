#!/bin/bash
# ncu --set full captures (one launch each) of tools/profile_iteration.py:
# NCU_SPECS="name:kernel_regex:skip ..."
mkdir -p gpurun_out
SPECS=${NCU_SPECS:-round_i8:k_round_i8:7 energy16:k_energy_tc:1 outer_i8:k_outer_i8:7 key_hist:k_key_hist:0 group_scatter:k_group_scatter:1 sum_tiles:k_sum_tiles:0 y_tiles:k_y_tiles:1}
for spec in $SPECS; do
  IFS=: read name rx skip <<< "$spec"
  timeout 900 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "iteration/" \
     -k regex:$rx -s $skip -c 1 -o gpurun_out/full_$name -f python tools/profile_iteration.py $PROFILE_ARGS > gpurun_out/ncu_$name.log 2>&1
  echo "$name: $(tail -1 gpurun_out/ncu_$name.log)"
done
