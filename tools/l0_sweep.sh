for l0 in 1e-6 1e-5 1e-4 1e-3; do
  export SBO_NS_L0=$l0
  timeout 300 python tools/profile_iteration.py > gpurun_out/l0_$l0.log 2>&1
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_l0.log 2>&1
  echo "l0=$l0 $(tail -1 gpurun_out/bench_l0.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['kernels']['k_polar_ns_cluster']['ms_per_step'], d['rmse'])") $(grep sweeps gpurun_out/l0_$l0.log | tr '\n' ' ')"
done
