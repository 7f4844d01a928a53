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

# dependent row loads after the row record: binary search with 3 record levels and a
# 4-wide parallel tail (today) vs aligned-sector B-tree separators (6 in the record)
def loads_binary(nn):
    ln = nn.copy()
    for _ in range(3):
        ln = ln // 2  # len after a level is either half or len-half-1 (<= half)
    extra = np.zeros_like(nn)
    while True:
        m = ln > 4
        if not m.any():
            break
        extra += m
        ln = np.where(m, ln // 2, ln)
    return extra + (ln > 0)


def loads_btree(nn, lo):
    a0 = (lo + 7) // 8 * 8
    hi = lo + nn
    m = np.maximum(0, (hi - a0 + 7) // 8)  # aligned separators in [lo, hi)
    lev = np.zeros_like(nn)
    top = m
    while True:
        big = top > 6
        if not big.any():
            break
        lev += big
        top = np.where(big, (top + 7) // 8, top)
    return lev + (nn > 0)


lo = off[rows]
lb, lt = loads_binary(n), loads_btree(n, lo)
print("mean loads after the record: binary", lb.mean(), " btree", lt.mean())
for k in range(0, 8):
    print(k, f"binary {100 * np.mean(lb == k):5.1f} %  btree {100 * np.mean(lt == k):5.1f} %")
for lim in (39, 48, 56, 79, 159, 319, 511, 1023):
    print(f"n <= {lim:4d}: {100 * np.mean(n <= lim):5.1f} %")
print("max n", n.max(), "max row", allrows.max())
