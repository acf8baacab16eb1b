#!/bin/bash
# Full GPU evidence: every -m gpu test, smoke, the sharded bench path on one GPU
# (gloo, functional), the default bench.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 > gpurun_out/pytest_gpu.log 2>&1
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
SBO_BENCH_ONE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 --m-total 1048576 --no-cpu-baseline --no-e2e > gpurun_out/bench_2r.log 2>&1
tail -c 300 gpurun_out/bench_2r.log; echo
if [ "${FULL_BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py > gpurun_out/bench.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'], d['e2e']['value'] if d.get('e2e') else None, d['roofline']['kernel'], d['phases_ms'])"
fi
if [ -n "$EXTRA_BENCH" ]; then
  timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $EXTRA_BENCH > gpurun_out/bench_extra.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_extra.log').read().strip().splitlines()[-1]); print('extra', d['config']['workload'][:50], d['value'], d['ms_per_step'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
fi
