bash tools/gpu_cand.sh
timeout 900 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_c.log 2>&1
python -c "import json; d=json.loads(open('gpurun_out/b_c.log').read().strip().splitlines()[-1]); print('C', d['value'], d['ms_per_step'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
