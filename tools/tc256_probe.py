"""p = 256 tensor-core pass on config-D-shaped data: flag rate, decisions vs the
float64 pass, and timing of one full representation."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1412_4944_b200 import signals  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402
from paper_1412_4944_b200.sbo import SboConfig, _init_into  # noqa: E402

m = int(os.environ.get("M", 1 << 18))
K = 32
dev = require_device()
rows = signals.unit_range(signals.patch_bytes(signals.scene(2048, 2048, 0), 16, m, 11))
eng = Engine(Signals.from_rows(rows, dev), 16, k_cap=K)
_init_into(eng, SboConfig(s0=16, k0=K, p0=4096, rounds=6, k_max=K, seed=1), m)
torch.cuda.synchronize()
res = {}
for tc in (True, False):
    eng.tc = tc
    if tc:
        eng.refresh_signals()
    for rep in range(2):
        torch.cuda.synchronize()
        t = time.perf_counter()
        eng.energy(0, K, False)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    res[tc] = (eng.state.best.clone(), eng.state.residual.clone(), dt,
               int(eng.flag_counts[-1].item()) if tc else 0)
b1, r1, t1, nf = res[True]
b0, r0, t0, _ = res[False]
print(f"m={m} K={K}: tc {t1*1e3:.1f} ms (flags {nf}, {100*nf/m:.2f}%), f64 {t0*1e3:.1f} ms, "
      f"decision mismatches {int((b1 != b0).sum().item())}")
