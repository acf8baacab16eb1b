mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none --nvtx --nvtx-include "iteration/" \
  -k regex:k_round_i8 -s 7 -c 1 -o gpurun_out/full_ri8 -f python tools/profile_iteration.py --m 1048576 --scene 2048 > gpurun_out/ncu_ri8.log 2>&1
tail -3 gpurun_out/ncu_ri8.log
