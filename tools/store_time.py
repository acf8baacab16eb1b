"""Throughput of codes persistence: device-streamed save_sbo_codes vs copy-to-host +
the reference's host writer (same bytes), at the bench workload size."""
import json
import os
import shutil
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, ".")
import paper_1412_4944_b200 as S  # noqa: E402
from paper_1412_4944_b200 import data, signals, store  # noqa: E402

m = int(os.environ.get("STORE_M", 1 << 20))
grid = signals.scene(2048, 2048, 0)
sig = data.extract_patches_device(grid, data.PatchConfig(patch_edge=8, count=m, seed=11))
rng = np.random.default_rng(0)
d = S.UnionDictionary([np.linalg.qr(rng.standard_normal((64, 64)))[0] for _ in range(16)])
dc = S.represent_device(sig, d, 8)
import torch  # noqa: E402
torch.cuda.synchronize()
res = {"m": m, "k": dc.k}
root = tempfile.mkdtemp(dir=os.environ.get("STORE_DIR", "/tmp"))
for name, fn in (("device_stream", lambda p: store.save_sbo_codes(p, dc)),
                 ("host_copy_then_write", lambda p: store.save_sbo_codes(p, dc.to_host()))):
    best = None
    for rep in range(3):
        path = os.path.join(root, f"{name}{rep}")
        t = time.perf_counter()
        fn(path)
        os.sync()
        dt = time.perf_counter() - t
        best = dt if best is None else min(best, dt)
        nbytes = os.path.getsize(os.path.join(path, "codes.odm"))
        shutil.rmtree(path)
    res[name] = {"s": best, "GB/s": nbytes / best / 1e9, "bytes": nbytes}
print(json.dumps(res))
shutil.rmtree(root)
