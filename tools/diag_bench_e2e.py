"""Run bench.run_e2e in isolation (optionally after a plain timed loop) to debug overlap."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1412_4944_b200.engine import Engine, Signals, require_device  # noqa: E402
from paper_1412_4944_b200.sbo import SboConfig, _block_rng, _init_into  # noqa: E402

os.environ["SBO_E2E_DEBUG"] = "1"
sys.argv = ["bench.py", "--steps", "4"]
a = bench.parse()
dev = require_device(0)
rows, m_total = bench.shard_signals(a, 0, 1)
eng = Engine(Signals.from_rows(rows, dev), a.s0, k_cap=a.K)
_init_into(eng, SboConfig(s0=8, k0=15, p0=4096, rounds=6, k_max=16, seed=1), m_total)
eng.represent_full()
torch.cuda.synchronize()
snap_blocks = eng.blocks.clone()
st = eng.state
snap = [t.clone() for t in (st.best, st.score, st.norm, st.residual, st.total)]
draws = _block_rng(1, 1, 15).standard_normal((72, 64))
if len(sys.argv) > 1 and os.environ.get("PRE") == "1":
    ent = eng.snapshot()
    for _ in range(3):
        eng.restore(ent)
        eng.iterate(m_total // 16, 6, draws)
print(bench.run_e2e(a, eng, rows, snap_blocks, snap, 15, m_total // 16, draws, None))
