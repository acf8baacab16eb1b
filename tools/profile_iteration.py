"""One SBO iteration inside an NVTX range, for ncu launch lists / captures.

    ncu --nvtx --nvtx-include "iteration/" --metrics gpu__time_duration.sum \
        --csv --log-file gpurun_out/launches.csv python tools/profile_iteration.py
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1412_4944_b200 import signals  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402
from paper_1412_4944_b200.sbo import SboConfig, _block_rng, _init_into  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1 << 24)
    ap.add_argument("--K", type=int, default=16)
    ap.add_argument("--iters", type=int, default=1)
    ap.add_argument("--p-edge", type=int, default=8)
    ap.add_argument("--s0", type=int, default=8)
    ap.add_argument("--scene", type=int, default=4096)
    a = ap.parse_args()
    dev = require_device()
    rows = signals.unit_range(signals.patch_bytes(signals.scene(a.scene, a.scene, 0), a.p_edge, a.m, 11))
    eng = Engine(Signals.from_rows(rows, dev), a.s0, k_cap=a.K)
    _init_into(eng, SboConfig(s0=a.s0, k0=a.K - 1, p0=4096, rounds=6, k_max=a.K, seed=1), a.m)
    eng.represent_full()
    torch.cuda.synchronize()
    draws = _block_rng(1, 1, eng.K).standard_normal((eng.p + 8, eng.p))
    K0 = eng.K
    snap = eng.blocks.clone()
    for _ in range(a.iters):
        eng.blocks.copy_(snap)
        eng.K = K0
        eng.represent_full()
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_push("iteration")
        out = eng.iterate(max(64, a.m // 16), 6, draws)
        torch.cuda.synchronize()
        torch.cuda.nvtx.range_pop()
    print("rmse", out.rmse, "flags", [int(f.item()) for f in eng.flag_counts[-3:]])
    print("jacobi sweeps new-block rounds:", eng.last_sweeps[0, :, 0].tolist())
    print("jacobi sweeps retrain (max over blocks):", eng.last_sweeps[1, :6].max(axis=1).tolist())


if __name__ == "__main__":
    main()
