#!/bin/bash
# correctness of the working build, then an A/B against libsbo_b200_base.so
timeout 300 python -m pytest tests/test_gpu_outer_i8.py tests/test_gpu_round_i8.py -x -q --timeout 120 2>&1 | tail -2
bash tools/ab.sh libsbo_b200_base.so libsbo_b200.so "$@"
