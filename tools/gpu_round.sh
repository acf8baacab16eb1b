#!/bin/bash
# One evidence session: parity tests, smoke, bench (both arms), ncu launch list,
# full ncu captures of the top kernels (NCU_SPECS name:regex:skip).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv python tools/profile_iteration.py > gpurun_out/launches.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 24 > gpurun_out/launch_summary.txt 2>&1
NCU_SPECS=${NCU_SPECS:-"round_retrain:k_round64:7 energy16:k_energy_tc:1 resid:k_round64:13 polar:k_polar_ns_cluster:6 init:k_init_block:0"} bash tools/gpu_prof.sh
tail -5 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log; tail -c 600 gpurun_out/bench.log; cat gpurun_out/launch_summary.txt
