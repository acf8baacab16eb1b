#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/tc_oracle_probe.py --m 1048576 > gpurun_out/tc_oracle_probe.log 2>&1; tail -1 gpurun_out/tc_oracle_probe.log
bash tools/config_sweep.sh
