#!/bin/bash
# Timing sweep over the other BASELINE configs at their stated sizes
# (informational, not bench lines): E = s0 in {4,8,16,32} x K in {4,16,64} at
# p = 64, m = 2^22; D = p 256, K 32, s0 16, m = 2^22.
mkdir -p gpurun_out
out=gpurun_out/config_sweep.jsonl; : > $out
run() { timeout 1200 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>>gpurun_out/sweep_err.log | tail -1 >> $out || echo "{\"failed\": \"$*\"}" >> $out; }
for K in 4 16 64; do for s0 in 4 8 16 32; do run --K $K --s0 $s0 --m-total 4194304; done; done
run --p-edge 16 --K 32 --s0 16 --m-total 4194304 --scene 4096
python - <<'PY'
import json
for l in open("gpurun_out/config_sweep.jsonl"):
    try:
        d = json.loads(l)
    except Exception:
        print("bad", l[:200]); continue
    if "failed" in d: print(d); continue
    print(d["config"]["workload"][:60], f"{d['value']:.3e}", f"{d['ms_per_step']:.2f} ms", d["phases_ms"])
PY
