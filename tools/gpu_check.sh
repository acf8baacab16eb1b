set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 900 python -m pytest tests -m gpu -q -rf --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1 || true
timeout 600 python bench.py --steps 3 --warmup 2 > gpurun_out/bench.log 2>&1 || true
tail -5 gpurun_out/pytest_gpu.log; tail -3 gpurun_out/smoke.log; tail -c 3000 gpurun_out/bench.log
