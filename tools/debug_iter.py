"""Time each ABI call of one iteration (synchronizing after every call) at a given m."""
import argparse
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1412_4944_b200 import _lib as L  # noqa: E402
from paper_1412_4944_b200 import signals  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402
from paper_1412_4944_b200.sbo import SboConfig, _block_rng, _init_into  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--m", type=int, default=1 << 16)
ap.add_argument("--K", type=int, default=16)
a = ap.parse_args()
dev = require_device()
orig = L.call
stats = {}


def timed(name, *args):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = orig(name, *args)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    s = stats.setdefault(name, [0, 0.0])
    s[0] += 1
    s[1] += dt
    if dt > 0.5:
        print(f"slow call {name}: {dt:.2f}s", flush=True)
    return r


L.call = timed
rows = signals.unit_range(signals.patch_bytes(signals.scene(2048, 2048, 0), 8, a.m, 11))
eng = Engine(Signals.from_rows(rows, dev), 8, k_cap=a.K)
print("init...", flush=True)
_init_into(eng, SboConfig(s0=8, k0=a.K - 1, p0=4096, rounds=6, k_max=a.K, seed=1), a.m)
print("represent...", flush=True)
eng.represent_full()
print("iterate...", flush=True)
out = eng.iterate(max(64, a.m // 16), 6, _block_rng(1, 1, eng.K).standard_normal((72, 64)))
print("rmse", out.rmse, flush=True)
for k, (n, t) in sorted(stats.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:28s} {n:5d} {t * 1e3:10.2f} ms")
