#!/bin/bash
# p = 256 integer-digit projection: its GPU tests, the p = 256 parity tests, and
# an A/B of SBO_CI8 on config D at m = 2^22 (bench, no profiler).
mkdir -p gpurun_out
make -s -j8 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_coef_i8.py -x -q > gpurun_out/pytest_ci8.log 2>&1
tail -3 gpurun_out/pytest_ci8.log
timeout 1200 python -m pytest tests -m gpu -q -k "256 or D or reference_suite" > gpurun_out/pytest_ci8_p256.log 2>&1
tail -3 gpurun_out/pytest_ci8_p256.log
bash tools/ab_env.sh SBO_CI8 1 0 --p-edge 16 --K 32 --s0 16 --m-total 4194304 --scene 4096
