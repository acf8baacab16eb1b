"""Bisect which part of bench.run_e2e serialises the signal upload with the step."""
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
copied = [torch.cuda.Event(), torch.cuda.Event()]
freed = [None, None]


def run(name, events, switch, refresh):
    def upload(j):
        with torch.cuda.stream(copier):
            if events and freed[j] is not None:
                copier.wait_event(freed[j])
            ybuf[j].copy_(host_y, non_blocking=True)
            copied[j].record(copier)

    def step(j):
        if events:
            compute.wait_event(copied[j])
        if switch:
            eng.sig.y = ybuf[j]
        if refresh:
            eng.refresh_signals()
        eng.restore(snap)
        eng.iterate(m // 16, 6, ddraws)
        if events:
            freed[j] = torch.cuda.Event()
            freed[j].record(compute)

    with torch.cuda.stream(compute):
        upload(0)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i in range(4):
            upload((i + 1) % 2)
            step(i % 2)
        torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t) / 4 * 1e3:.2f} ms/step", flush=True)
    eng.sig.y = ybuf[0]


run("plain", False, False, False)
run("events", True, False, False)
run("switch", False, True, False)
run("refresh", False, False, True)
run("all", True, True, True)

host_blocks = snap["blocks"][:15].cpu().pin_memory()
host_state = [t.cpu().pin_memory() for t in snap["state"]]
host_draws = torch.from_numpy(np.ascontiguousarray(draws)).pin_memory()
dev_draws = torch.empty(host_draws.shape, dtype=torch.float64, device=dev)
out_blocks = torch.empty((16, 64, 64), dtype=torch.float64).pin_memory()
out_best = torch.empty(m, dtype=torch.int32).pin_memory()
out_res = torch.empty(m, dtype=torch.float64).pin_memory()
st = eng.state


def run2(name, stage, d2h):
    def upload(j):
        with torch.cuda.stream(copier):
            if freed[j] is not None:
                copier.wait_event(freed[j])
            ybuf[j].copy_(host_y, non_blocking=True)
            copied[j].record(copier)

    def stage_state():
        eng.blocks[:15].copy_(host_blocks, non_blocking=True)
        for dst, src in zip((st.best, st.score, st.norm, st.residual, st.total), host_state):
            dst.copy_(src, non_blocking=True)
        dev_draws.copy_(host_draws, non_blocking=True)

    def step(j):
        compute.wait_event(copied[j])
        eng.sig.y = ybuf[j]
        eng.refresh_signals()
        if stage:
            eng.K = 15
            eng.exact_scores = True
        else:
            eng.restore(snap)
        eng.iterate(m // 16, 6, dev_draws if stage else ddraws)
        if d2h:
            out_blocks.copy_(eng.blocks[:16], non_blocking=True)
            out_best.copy_(st.best, non_blocking=True)
            out_res.copy_(st.residual, non_blocking=True)
        freed[j] = torch.cuda.Event()
        freed[j].record(compute)

    with torch.cuda.stream(compute):
        upload(0)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for i in range(4):
            if stage:
                stage_state()
            upload((i + 1) % 2)
            step(i % 2)
        torch.cuda.synchronize()
    print(f"{name}: {(time.perf_counter() - t) / 4 * 1e3:.2f} ms/step", flush=True)
    eng.sig.y = ybuf[0]


run2("restore, no d2h", False, False)
run2("restore, d2h", False, True)
run2("stage, no d2h", True, False)
run2("stage, d2h", True, True)
