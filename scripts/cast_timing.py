"""A/B timing of the batched cast kernel on the bench workload (config 3),
for comparing kernel variants built with different defines:

    RL_CDDT_LIB=paper_1705_01167_b200/librl_cddt_minb4.so python scripts/cast_timing.py
Prints one JSON line: ms per 100M-query launch and an output checksum.
"""
import hashlib
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_01167_b200 as rl  # noqa: E402
from paper_1705_01167_b200 import synth  # noqa: E402

n = int(os.environ.get("NQ", 100_000_000))
cfg = os.environ.get("CFG", "3")
if cfg == "3":
    g, K, mr, prune = synth.polygon_map(4000, 4000, 0.12, seed=3), 200, 1000.0, True
elif cfg == "2":
    g, K, mr, prune = synth.maze_map(), 120, 500.0, False
else:
    g, K, mr, prune = synth.rect_map(), 108, 300.0, False
c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(mr, K), prune=prune)
qx, qy, qt = synth.free_queries(g, n, seed=7)
if os.environ.get("SORT") == "theta":  # locality experiment: queries ordered by direction
    o = np.argsort(qt, kind="stable")
    qx, qy, qt = qx[o], qy[o], qt[o]
elif os.environ.get("SORT") == "chunk":  # ordered by direction within 8M-query chunks
    ch = 8_000_000
    for s0 in range(0, n, ch):
        o = np.argsort(qt[s0:s0 + ch], kind="stable") + s0
        qx[s0:s0 + ch], qy[s0:s0 + ch], qt[s0:s0 + ch] = qx[o], qy[o], qt[o]
dx, dy, dt = (torch.from_numpy(a).cuda() for a in (qx, qy, qt))
out = torch.empty_like(dx)
for _ in range(3):
    c.cast_batch(dx, dy, dt, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = int(os.environ.get("REPS", 10))
e0.record()
for _ in range(reps):
    c.cast_batch(dx, dy, dt, out=out)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
h = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]
print(json.dumps(dict(lib=os.environ.get("RL_CDDT_LIB", "default"), cfg=cfg, n=n, ms=ms,
                      gcasts_per_s=n / ms / 1e6, sha=h)))
