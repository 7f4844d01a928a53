"""Config-1 small-batch timing (500x500 rects, theta_disc 108, max_range 300,
100k queries): Python-loop calls, CUDA-graph replay of the same calls, and
single-launch latency. python scripts/small_batch.py [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_01167_b200 as rl  # noqa: E402
from paper_1705_01167_b200 import synth  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
g = synth.rect_map()
c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(300.0, 108), device=0)
qx, qy, qt = (torch.from_numpy(a).cuda() for a in synth.free_queries(g, 100_000, seed=7))
o = torch.empty_like(qx)


def ev(fn, n):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / n * 1e3  # us


for _ in range(5):
    c.cast_batch(qx, qy, qt, out=o)
ref = o.clone()
res = {"loop_us": ev(lambda: c.cast_batch(qx, qy, qt, out=o), reps)}
lat = []
for _ in range(50):
    lat.append(ev(lambda: c.cast_batch(qx, qy, qt, out=o), 1))
res["single_launch_us_p50"] = float(np.median(lat))
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    c.cast_batch(qx, qy, qt, out=o)
torch.cuda.current_stream().wait_stream(s)
gr = torch.cuda.CUDAGraph()
per_graph = 20
with torch.cuda.graph(gr):
    for _ in range(per_graph):
        c.cast_batch(qx, qy, qt, out=o)
gr.replay()
torch.cuda.synchronize()
assert torch.equal(o, ref)
res["graph_us_per_batch"] = ev(gr.replay, max(1, reps // per_graph)) / per_graph
res["graph_casts_per_s"] = 100_000 / res["graph_us_per_batch"] * 1e6
print(res)
