#!/bin/bash
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_scale.py tests/test_gpu_tc256.py -x -q --timeout 600 2>&1 | tail -3
EXTRA_BENCH="--K 64 --s0 16 --m-total 4194304" bash -c 'timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --K 64 --s0 16 --m-total 4194304 > gpurun_out/bench_k64.log 2>&1'
python -c "import json; d=json.loads(open('gpurun_out/bench_k64.log').read().strip().splitlines()[-1]); print('K64 s0 16', d['value'], d['ms_per_step'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --K 64 --s0 8 --m-total 4194304 > gpurun_out/bench_k64b.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/bench_k64b.log').read().strip().splitlines()[-1]); print('K64 s0 8', d['value'], d['ms_per_step'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
timeout 900 python tools/tc_oracle_probe.py --m 1048576 | tail -1
