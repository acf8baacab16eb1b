#!/bin/bash
# new-block chain evidence at config B (m = 2^20): sweeps, launch list, ncu of k_init_block / polar
mkdir -p gpurun_out
python tools/profile_iteration.py --m 1048576 --scene 2048 > gpurun_out/chain_run.log 2>&1
timeout 300 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/chain_launches.csv python tools/profile_iteration.py --m 1048576 --scene 2048 \
  > gpurun_out/chain_ncu.log 2>&1
for k in k_init_block k_polar_ns_cluster; do
  timeout 300 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "iteration/" \
    -k regex:$k -c 1 -o gpurun_out/full_$k -f python tools/profile_iteration.py --m 1048576 --scene 2048 \
    > gpurun_out/ncu_$k.log 2>&1
done
tail -3 gpurun_out/chain_run.log
