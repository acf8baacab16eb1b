#!/bin/bash
# init Jacobi rotation A/B at config B (SBO_INIT_LP = -8: IEEE rotation, 8: fast rotation), then the init tests
mkdir -p gpurun_out
for rep in 1 2; do
for lp in -8 8; do
  SBO_INIT_LP=$lp timeout 300 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/rot_$lp.csv \
    python tools/profile_iteration.py --m 1048576 --scene 2048 > gpurun_out/rot_$lp.log 2>&1
  echo "LP=$lp rep $rep: $(grep 'new-block' gpurun_out/rot_$lp.log) $(python tools/launch_summary.py gpurun_out/rot_$lp.csv | grep init_block)"
done
done
timeout 600 python -m pytest tests/test_gpu_polar_cluster.py tests/test_gpu_parity.py -q -x 2>&1 | tail -2
