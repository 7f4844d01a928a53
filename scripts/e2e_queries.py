"""Config-3 end-to-end timing of rl_cddt_cast_queries_host (an array of RayQuery
{double x, y, theta} in host memory -> double ranges), pageable and pinned:
    python scripts/e2e_queries.py"""
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

n = int(os.environ.get("NQ", 50_000_000))
g, qx, qy, qt, _ = bench.make_workload(n, 0)
c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(1000.0, 200), prune=True)
q = np.stack([a.numpy().astype(np.float64) for a in (qx, qy, qt)], axis=1)
res = {}
for kind in ("pinned", "pageable"):
    if kind == "pinned":
        hq = torch.from_numpy(q).pin_memory().numpy()
        ho = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
    else:
        hq, ho = q, np.zeros(n)
    c.cast_queries(hq, out=ho)
    t0 = time.perf_counter()
    for _ in range(3):
        c.cast_queries(hq, out=ho)
    ms = (time.perf_counter() - t0) / 3 * 1e3
    res[kind] = dict(ms=ms, gcasts_per_s=n / ms / 1e6, checksum=float(ho.sum()))
print(json.dumps(dict(n=n, bytes_per_query=32, **res)))
