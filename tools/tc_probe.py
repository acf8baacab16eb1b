"""GPU probe: tensor-core energy pass vs the exact float64 pass on the bench workload.

    python tools/tc_probe.py [--m 1048576] [--K 16]
Prints decision mismatches (must be 0), the flagged fraction, residual accuracy
and kernel timings.
"""
import argparse
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1412_4944_b200 import signals  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402
from paper_1412_4944_b200.sbo import SboConfig, _init_into  # noqa: E402


def timed(fn, reps=3):
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--m", type=int, default=1 << 20)
    ap.add_argument("--K", type=int, default=16)
    ap.add_argument("--s0", type=int, default=8)
    ap.add_argument("--kind", default="squared-sum")
    ap.add_argument("--gauss", action="store_true")
    a = ap.parse_args()
    dev = require_device()
    if a.gauss:
        rows = signals.gaussian_signals(64, a.m, seed=3)
    else:
        rows = signals.unit_range(signals.patch_bytes(signals.scene(2048, 2048, 0), 8, a.m, 11))
    os.environ["SBO_TC"] = "0"
    ref = Engine(Signals.from_rows(rows, dev), a.s0, a.kind, k_cap=a.K)
    t0 = time.time()
    _init_into(ref, SboConfig(s0=a.s0, k0=a.K, p0=4096, rounds=6, k_max=a.K, seed=1), a.m)
    torch.cuda.synchronize()
    print(f"init {time.time() - t0:.1f}s")
    t_f64 = timed(lambda: ref.energy(0, a.K, False), reps=1)
    os.environ["SBO_TC"] = "1"
    tc = Engine(Signals.from_rows(rows, dev), a.s0, a.kind, k_cap=a.K)
    tc.set_blocks(ref.blocks[: a.K])
    t_tc = timed(lambda: tc.energy(0, a.K, False))
    nflag = int(tc.nflag.item())
    # kernel-only timing (no recheck)
    def only_tc():
        tc.nflag.zero_()
        from paper_1412_4944_b200 import _lib as L
        s = tc.state
        L.call("sbo_tc_energy", tc.yh.data_ptr(), tc.yl.data_ptr(), tc.escale.data_ptr(), tc.m,
               tc.qh.data_ptr(), tc.ql.data_ptr(), tc.fscale.data_ptr(), 0, a.K, a.s0, tc.kind,
               0, s.best.data_ptr(), s.score.data_ptr(), s.residual.data_ptr(),
               tc.flags.data_ptr(), tc.nflag.data_ptr(), None, tc.stream)
    t_kernel = timed(only_tc)
    tc.energy(0, a.K, False)
    b_ref, b_tc = ref.state.best.cpu().numpy(), tc.state.best.cpu().numpy()
    r_ref, r_tc = ref.state.residual.cpu().numpy(), tc.state.residual.cpu().numpy()
    n_ref = ref.state.norm.cpu().numpy()
    mism = np.nonzero(b_ref != b_tc)[0]
    rel = np.abs(r_tc - r_ref) / np.maximum(r_ref, 1e-300)
    absn = np.abs(r_tc - r_ref) / np.maximum(n_ref, 1e-300)
    print(f"m={a.m} K={a.K} s0={a.s0} kind={a.kind} gauss={a.gauss}")
    print(f"f64 pass {t_f64:.2f} ms | tc pass+recheck {t_tc:.3f} ms | tc kernel {t_kernel:.3f} ms")
    flops = 2.0 * 64 * 64 * a.K * a.m
    print(f"tc kernel algorithmic {flops / t_kernel / 1e9:.1f} TFLOP/s (3 fp16 MMAs each)")
    print(f"flagged {nflag} ({nflag / a.m:.2e}); decision mismatches after recheck: {mism.size}")
    print(f"residual rel err: median {np.median(rel):.2e} p99 {np.quantile(rel, 0.99):.2e} "
          f"max {rel.max():.2e}; |dR|/||y||^2 max {absn.max():.2e}")
    print(f"residual/||y||^2: median {np.median(r_ref / n_ref):.2e} min {np.min(r_ref / n_ref):.2e}")
    # incremental: drop the last block, then add it back incrementally
    ref2 = ref
    ref2.energy(0, a.K - 1, False)
    ref2.energy(a.K - 1, a.K, True)
    tc.energy(0, a.K - 1, False)
    tc.energy(a.K - 1, a.K, True)
    mi = np.nonzero(ref2.state.best.cpu().numpy() != tc.state.best.cpu().numpy())[0]
    print(f"incremental: flagged {int(tc.nflag.item())}, mismatches {mi.size}")
    print("block sizes", np.bincount(b_ref, minlength=a.K))


if __name__ == "__main__":
    main()
