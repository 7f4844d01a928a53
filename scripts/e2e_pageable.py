"""Config-3 end-to-end timing through the host-pointer C ABI with PAGEABLE host
buffers (plain numpy arrays, what a reference caller holds) beside pinned ones:
    python scripts/e2e_pageable.py"""
import hashlib
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1705_01167_b200 as rl  # noqa: E402

n = int(os.environ.get("NQ", 100_000_000))
g, qx, qy, qt, _ = bench.make_workload(n, 0)
c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(1000.0, 200), prune=True)
res = {}
for kind in ("pinned", "pageable"):
    if kind == "pinned":
        hx, hy, ht = qx.numpy(), qy.numpy(), qt.numpy()
        ho = torch.empty(n, dtype=torch.float32).pin_memory().numpy()
    else:
        hx, hy, ht = (np.array(a.numpy(), copy=True) for a in (qx, qy, qt))
        ho = np.zeros(n, dtype=np.float32)
    c.cast_batch(hx, hy, ht, out=ho)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        c.cast_batch(hx, hy, ht, out=ho)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / 3 * 1e3
    res[kind] = dict(ms=ms, gcasts_per_s=n / ms / 1e6, sha=hashlib.sha256(ho.tobytes()).hexdigest()[:16])
print(json.dumps(dict(lib=os.environ.get("RL_CDDT_LIB", "default"), n=n, **res)))
