#!/bin/bash
# A/B of the new-block chain kernels (Jacobi lanes per pair, Newton-Schulz cluster size) at config B,
# then the GPU test suite.
mkdir -p gpurun_out
for cfg in "16 4" "4 4" "4 8" "8 0" "4 0"; do
  set -- $cfg
  SBO_INIT_LP=$1 SBO_NS_CLUSTER=$2 timeout 300 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum \
    --clock-control none --csv --log-file gpurun_out/chainab_$1_$2.csv \
    python tools/profile_iteration.py --m 1048576 --scene 2048 > gpurun_out/chainab_$1_$2.log 2>&1
  echo "== LP=$1 NC=$2"; tail -2 gpurun_out/chainab_$1_$2.log
  python tools/launch_summary.py gpurun_out/chainab_$1_$2.csv | grep -E "init_block|polar_ns|total"
done
for X in "16 4" "4 0"; do
  set -- $X
  for rep in 1 2; do
    SBO_INIT_LP=$1 SBO_NS_CLUSTER=$2 timeout 300 python bench.py --m-total 1048576 --scene 2048 --steps 10 --warmup 3 \
      --no-cpu-baseline --no-e2e > gpurun_out/chainab_bench_$1_$2.$rep.log 2>&1
    python -c "
import json,sys; d=json.loads(open('gpurun_out/chainab_bench_$1_$2.$rep.log').read().strip().splitlines()[-1])
print('bench B LP=$1 NC=$2', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['phases_ms'].items()})"
  done
done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/chainab_pytest.log 2>&1; tail -3 gpurun_out/chainab_pytest.log
