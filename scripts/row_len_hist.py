"""Distribution of the searched row length n over config-3 queries (PCDDT):
how many search levels the per-row records cover. python scripts/row_len_hist.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_01167_b200 as rl  # noqa: E402
from paper_1705_01167_b200 import synth  # noqa: E402

g = synth.polygon_map(4000, 4000, 0.12, seed=3)
c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(1000.0, 200), prune=True)
q = [torch.from_numpy(a.astype(np.float64)).cuda() for a in synth.free_queries(g, 1_000_000, seed=7)]
rr = torch.empty(q[0].numel(), dtype=torch.int64, device="cuda")
ri = torch.empty(q[0].numel(), dtype=torch.int32, device="cuda")
c.cast_batch_f64(*q, res_row=rr, res_idx=ri)
torch.cuda.synchronize()
e = c.export()
off = e["row_off"].astype(np.int64)
rows = rr.cpu().numpy()
rows = rows[rows >= 0]
n = off[rows + 1] - off[rows]
print("resolved queries", rows.size)
for lim in (1, 3, 7, 15, 31, 63, 127, 255):
    print(f"n <= {lim:4d}: {100 * np.mean(n <= lim):5.1f} %")
print("mean n", n.mean(), "median", np.median(n), "p90", np.percentile(n, 90))
allrows = off[1:] - off[:-1]
print("all rows: mean", allrows.mean(), "median", np.median(allrows))
