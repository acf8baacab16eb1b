timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -2
for s0 in 16 32; do timeout 600 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --K 16 --s0 $s0 --m-per-gpu 4194304 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['s0'], d['value'], d['ms_per_step'])"; done
