#!/bin/bash
# Final evidence of the round at HEAD: every GPU test, smoke, both bench arms,
# the config-C launch list, ncu --set full of the three top kernels.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], 'e2e', d['e2e']['value'], 'ingest', d['e2e_ingest']['value'], d['clocks'])"
timeout 900 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/launches.csv python tools/profile_iteration.py > gpurun_out/launches.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 30 > gpurun_out/launch_summary.txt 2>&1; head -6 gpurun_out/launch_summary.txt
NCU_SPECS="round_i8:k_round_i8:7 energy16:k_energy_tc:1 outer_i8:k_outer_i8:7" bash tools/gpu_ncu.sh
# config D (p = 256) at its stated m = 2^22: a bench line and the launch list
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --p-edge 16 --K 32 --s0 16 --m-total 4194304 --scene 4096 > gpurun_out/bench_D.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_D.log').read().strip().splitlines()[-1]); print('bench D', d['value'], d['ms_per_step'], d['phases_ms'])"
DM=4194304 bash tools/gpu_d_launches.sh > gpurun_out/launches_D22_summary.txt 2>&1; head -8 gpurun_out/launches_D22_summary.txt
