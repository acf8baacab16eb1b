"""GPU probe: the full representation (tcgen05 energy pass with its certificate and
float64 re-decision, then the integer-digit residual pass) against the CPU oracle
(oracle.code_signals, the restatement of sbo.py:138-220) on the bench workload.

    python tools/tc_oracle_probe.py [--m 1048576] [--K 16] [--s0 8]

Prints one JSON line: decision mismatches (must be 0 outside float64 near-ties),
the flagged fraction, and the residual / energy accuracy.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import sbo_oracle as O  # noqa: E402
from paper_1412_4944_b200 import signals  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402
from paper_1412_4944_b200.sbo import SboConfig, _init_into  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1 << 20)
    ap.add_argument("--K", type=int, default=16)
    ap.add_argument("--s0", type=int, default=8)
    ap.add_argument("--scene", type=int, default=4096)
    a = ap.parse_args()
    dev = require_device()
    rows = signals.unit_range(signals.patch_bytes(signals.scene(a.scene, a.scene, 0), 8, a.m, 11))
    eng = Engine(Signals.from_rows(rows, dev), a.s0, k_cap=a.K)
    _init_into(eng, SboConfig(s0=a.s0, k0=a.K, p0=4096, rounds=6, k_max=a.K, seed=1), a.m)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.represent_full()
    torch.cuda.synchronize()
    t_gpu = time.perf_counter() - t0
    best = eng.state.best.cpu().numpy().astype(np.int64)
    res = eng.state.residual.cpu().numpy()
    flagged = int(eng.flag_counts[-1].item()) if eng.flag_counts else 0
    blocks = list(eng.blocks[: a.K].cpu().numpy())
    y = rows.T.astype(np.float64)
    t0 = time.perf_counter()
    rep = O.code_signals(y, blocks, a.s0, workers=os.cpu_count() or 1)
    t_cpu = time.perf_counter() - t0
    diff = np.nonzero(best != rep.block)[0]
    # float64 energy gap of each mismatch (a documented near-tie when < 1e-12 rel)
    gaps = []
    for j in diff[:64]:
        e = [O.energy_of(y[:, j], q, a.s0) for q in (blocks[best[j]], blocks[rep.block[j]])]
        gaps.append(abs(e[0] - e[1]) / max(abs(e[1]), 1e-300))
    n2 = (y ** 2).sum(axis=0)
    out = {"m": a.m, "K": a.K, "s0": a.s0, "mismatches": int(diff.size),
           "mismatch_max_rel_gap": max(gaps) if gaps else None,
           "flagged_fraction": flagged / a.m,
           "residual_max_abs_err_over_norm2": float(np.max(np.abs(res - rep.residual_sq) /
                                                           np.maximum(n2, 1e-300))),
           "gpu_represent_s": t_gpu, "cpu_oracle_s": t_cpu,
           "oracle": "oracle.code_signals (numpy/OpenBLAS float64, sbo.py:138-220)"}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
