#!/bin/bash
# A/B of the tensor-core certificate constant (base build vs working build) at config C, flag counts
mkdir -p gpurun_out
for L in libsbo_b200_base.so libsbo_b200.so; do
  SBO_LIB=$L timeout 600 python tools/profile_iteration.py > gpurun_out/coef_$L.log 2>&1; echo "$L $(head -1 gpurun_out/coef_$L.log)"
done
bash tools/ab.sh libsbo_b200_base.so libsbo_b200.so
timeout 900 python -m pytest tests/test_gpu_bench_scale.py tests/test_gpu_parity.py -x -q > gpurun_out/coef_pytest.log 2>&1; tail -2 gpurun_out/coef_pytest.log
