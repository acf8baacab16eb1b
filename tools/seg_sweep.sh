for sl in ${SEGS:-1024 896 1024 896}; do
  export SBO_SEG_LEN=$sl
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_sl.log 2>&1
  echo "seg=$sl $(tail -1 gpurun_out/bench_sl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print(d['ms_per_step'], k['k_round64']['ms_per_step'], k['k_round64<resid>']['ms_per_step'], d['rmse'])")"
done
