"""Config A through the public API: sbo_train(k0=4 -> k_max=14) on the desk fixture,
timed on the device path (the reference takes ~4.7 s on 8 cores)."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1412_4944_b200 as S  # noqa: E402

d = np.load(Path(__file__).resolve().parents[1] / "tests" / "golden" / "desk_patches.npz")
y = (d["u8"].astype(np.float64) / 255.0).astype(np.float32).T.astype(np.float64)
cfg = S.SboConfig(s0=8, k0=4, p0=4096, rounds=6, k_max=14, seed=1)
S.sbo_train(y, cfg)  # warm-up (library load, kernel attributes)
t = time.perf_counter()
dic, code, a, rep = S.sbo_train(y, cfg)
dt = time.perf_counter() - t
print(f"config A sbo_train: {dt:.3f} s wall, K={len(dic.blocks)}, rmse={rep.rows[-1].rmse:.6f}"
      if hasattr(rep, "rows") else f"config A sbo_train: {dt:.3f} s wall, K={len(dic.blocks)}")
