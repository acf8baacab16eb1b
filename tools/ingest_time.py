"""Time device patch extraction (data.extract_rows) at the bench workload size."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1412_4944_b200 import data, signals  # noqa: E402

m = 1 << 20
grid = signals.scene(2048, 2048, 0)
r, c = data.patch_corners(2048, 2048, 8, m, 11)
dev = torch.device("cuda", 0)
g, code = data.upload_grid(grid, dev)
rd = torch.from_numpy(r.astype(np.int32)).to(dev)
cd = torch.from_numpy(c.astype(np.int32)).to(dev)
for dt, norm in ((torch.float32, "unit-range"), (torch.float64, "unit-range"),
                 (torch.float64, "unit-range-dc-removed")):
    out = torch.empty((m, 64), dtype=dt, device=dev)
    for _ in range(3):
        data.extract_rows(g, code, 8, rd, cd, norm, out=out)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        data.extract_rows(g, code, 8, rd, cd, norm, out=out)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"{dt} {norm}: {ms * 1e3:.1f} us, {out.numel() * out.element_size() / ms / 1e6:.0f} GB/s written")
