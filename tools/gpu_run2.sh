set -x
./tools/fp64_micro > gpurun_out/fp64_micro.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_iteration.py > gpurun_out/launches.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv 20 > gpurun_out/launch_summary.txt 2>&1
NCU_SPECS="round_retrain:k_round_f64:6 round_resid:k_round_f64:12 init_block:k_init_block:0 polar_retrain:k_polar_ns:6" bash tools/gpu_prof.sh
cat gpurun_out/fp64_micro.txt; tail -3 gpurun_out/pytest_gpu.log; tail -c 1500 gpurun_out/bench.log; cat gpurun_out/launch_summary.txt
