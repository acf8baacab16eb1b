#!/bin/bash
# Timing sweep over the other BASELINE configs (informational, not bench lines).
mkdir -p gpurun_out
out=gpurun_out/config_sweep.jsonl; : > $out
run() { timeout 900 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e "$@" 2>gpurun_out/sweep_err.log | tail -1 >> $out || echo "{\"failed\": \"$*\"}" >> $out; }
run --K 4 --s0 8 --m-per-gpu 4194304
run --K 16 --s0 4 --m-per-gpu 4194304
run --K 16 --s0 16 --m-per-gpu 4194304
run --K 16 --s0 32 --m-per-gpu 4194304
run --K 64 --s0 8 --m-per-gpu 4194304
run --K 16 --s0 8 --m-per-gpu 16777216
run --p-edge 16 --K 32 --s0 16 --m-per-gpu 1048576
python - <<'PY'
import json
for l in open("gpurun_out/config_sweep.jsonl"):
    try:
        d = json.loads(l)
    except Exception:
        print("bad", l[:200]); continue
    if "failed" in d: print(d); continue
    print(d["config"]["workload"][:90], f"{d['value']:.3e}", f"{d['ms_per_step']:.2f} ms")
PY
