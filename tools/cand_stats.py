"""Candidate-block statistics of the float64 re-decision after the 16-block
tensor-core pass: flagged signals, candidates per signal, union per 64-signal tile."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1412_4944_b200 import signals  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402
from paper_1412_4944_b200.sbo import SboConfig, _init_into  # noqa: E402

m = 1 << 20
dev = require_device()
rows = signals.unit_range(signals.patch_bytes(signals.scene(2048, 2048, 0), 8, m, 11))
eng = Engine(Signals.from_rows(rows, dev), 8, k_cap=16)
_init_into(eng, SboConfig(s0=8, k0=16, p0=4096, rounds=6, k_max=16, seed=1), m)
eng.energy(0, 16, False)
torch.cuda.synchronize()
n = int(eng.nflag.item())
cand = eng.cand_sorted[:n].cpu().numpy().astype(np.uint32)
pc = np.array([bin(int(c)).count("1") for c in cand])
unions = []
for t in range(0, n, 64):
    u = np.bitwise_or.reduce(cand[t:t + 64])
    unions.append(bin(int(u)).count("1"))
unions = np.array(unions)
print(f"flagged {n} ({100 * n / m:.2f}%), candidates per signal mean {pc.mean():.2f} max {pc.max()}, "
      f"union per 64-tile mean {unions.mean():.2f} (pairs {pc.sum()}, tile-block passes {unions.sum() * 64})")
