"""A/B timing of small range-only batches (config 1: 100 k queries on the
500x500 map; config 5's 1 M queries on the 2000x2000 maze, theta_disc 108):
ms per batch back to back, single-batch latency, and an output checksum.
RL_CDDT_LIB / RL_CAST_COOP select the variant."""
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


def ev(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


res = {"lib": os.environ.get("RL_CDDT_LIB", "default"), "coop": os.environ.get("RL_CAST_COOP", "1")}
for name, g, K, mr, nq in (("cfg1", synth.rect_map(), 108, 300.0, 100_000),
                           ("cfg5q", synth.maze_map(), 108, 0.0, 1_000_000)):
    c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(mr, K))
    q = [torch.from_numpy(a).cuda() for a in synth.free_queries(g, nq, seed=31)]
    o = torch.empty_like(q[0])
    res[name + "_ms"] = ev(lambda: c.cast_batch(*q, out=o), 100)
    res[name + "_lat_ms"] = float(np.median([ev(lambda: c.cast_batch(*q, out=o), 1) for _ in range(30)]))
    res[name + "_sha"] = hashlib.sha256(o.cpu().numpy().tobytes()).hexdigest()[:12]
print(json.dumps(res))
