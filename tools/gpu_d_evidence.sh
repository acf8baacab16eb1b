#!/bin/bash
# Config D evidence: the config sweep (E + D at 2^22), the D launch list at 2^22,
# ncu --set full of the p = 256 kernels at 2^20 (summaries via tools/ncu_summary.py).
mkdir -p gpurun_out
make -s -j8 > /dev/null 2>&1
bash tools/config_sweep.sh
DM=4194304 bash tools/gpu_d_launches.sh > gpurun_out/launches_D22_summary.txt 2>&1
NCU_SPECS="coef_i8:k_coef_i8:7 select_coded:k_select_coded:7 outer_sparse:k_outer_sparse256:7 energy256:k_energy_tc256:1 q_digits256:k_q_digits256:3" \
PROFILE_ARGS="--m 1048576 --scene 4096 --p-edge 16 --K 32 --s0 16" bash tools/gpu_ncu.sh
