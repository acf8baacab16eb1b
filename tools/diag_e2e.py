"""Diagnose the e2e step: compute-only vs pipelined upload vs upload-only."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1412_4944_b200 import signals  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402
from paper_1412_4944_b200.sbo import SboConfig, _block_rng, _init_into  # noqa: E402

dev = require_device()
m = 1 << 20
rows = signals.unit_range(signals.patch_bytes(signals.scene(2048, 2048, 0), 8, m, 11))
eng = Engine(Signals.from_rows(rows, dev), 8, k_cap=16)
_init_into(eng, SboConfig(s0=8, k0=15, p0=4096, rounds=6, k_max=16, seed=1), m)
eng.represent_full()
snap = eng.snapshot()
draws = _block_rng(1, 1, 15).standard_normal((72, 64))
ddraws = torch.from_numpy(draws).to(dev)
host_y = torch.from_numpy(rows).pin_memory()
compute, copier = torch.cuda.Stream(), torch.cuda.Stream()
ybuf = [eng.sig.y, torch.empty_like(eng.sig.y)]


def timed(fn, n=4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(n):
        fn(i)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / n * 1e3


def only0(i):
    eng.restore(snap)
    t0 = time.perf_counter()
    eng.iterate(m // 16, 6, draws)
    if i == 0:
        print("   default stream: host time in iterate", (time.perf_counter() - t0) * 1e3)


print("compute only, default stream ms", timed(only0))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
only0(1)
e1.record()
torch.cuda.synchronize()
print("  event-timed", e0.elapsed_time(e1))
with torch.cuda.stream(compute):
    def only(i):
        eng.restore(snap)
        eng.iterate(m // 16, 6, draws)
    print("compute only ms", timed(only))

    def up_only(i):
        with torch.cuda.stream(copier):
            ybuf[i % 2].copy_(host_y, non_blocking=True)
    print("upload only ms", timed(up_only))

    def both(i):
        eng.restore(snap)
        with torch.cuda.stream(copier):
            ybuf[(i + 1) % 2].copy_(host_y, non_blocking=True)
        t0 = time.perf_counter()
        eng.iterate(m // 16, 6, ddraws)
        print("   host time in iterate", (time.perf_counter() - t0) * 1e3)
    print("both ms", timed(both))

host_blocks = snap["blocks"].cpu().pin_memory()
host_state = [t.cpu().pin_memory() for t in snap["state"]]
out_res = torch.empty(m, dtype=torch.float64).pin_memory()
st = eng.state
with torch.cuda.stream(compute):
    def v_state(i):
        eng.blocks.copy_(host_blocks, non_blocking=True)
        for dst, src in zip((st.best, st.score, st.norm, st.residual, st.total), host_state):
            dst.copy_(src, non_blocking=True)
        eng.K = 15
        with torch.cuda.stream(copier):
            ybuf[(i + 1) % 2].copy_(host_y, non_blocking=True)
        eng.iterate(m // 16, 6, ddraws)
    print("H2D state + upload ms", timed(v_state))

    def v_split(i):
        eng.restore(snap)
        with torch.cuda.stream(copier):
            ybuf[(i + 1) % 2].copy_(host_y, non_blocking=True)
        eng.refresh_signals()
        eng.iterate(m // 16, 6, ddraws)
    print("split + upload ms", timed(v_split))

    def v_d2h(i):
        eng.restore(snap)
        with torch.cuda.stream(copier):
            ybuf[(i + 1) % 2].copy_(host_y, non_blocking=True)
        eng.iterate(m // 16, 6, ddraws)
        out_res.copy_(st.residual, non_blocking=True)
    print("D2H + upload ms", timed(v_d2h))
