"""Config-5 incremental-update timing: rounds of 50 random 3x3 edits on the
2000x2000 maze (theta_disc 108), host wall per round. python scripts/edit_timing.py [rounds]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_01167_b200 as rl  # noqa: E402
from paper_1705_01167_b200 import synth  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 30
g = synth.maze_map()
c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(0.0, 108), device=0)
times = []
for r in range(rounds):
    xy, occ = synth.block_edits(2000, 2000, 50, seed=9000 + r)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c.set_occupancy_batch(xy, occ)
    times.append(1e3 * (time.perf_counter() - t0))
print({"ms_per_round": [round(t, 3) for t in times], "p50": float(np.median(times)),
       "zero_points": c.zero_point_count()})
