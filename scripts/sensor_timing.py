"""Config-2 sensor-update timing (2,500 particles x 61 beams, 2000x2000 maze,
501x501 table): python scripts/sensor_timing.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

print(bench.other_configs.__doc__ and "", end="")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_01167_b200 as rl  # noqa: E402
from paper_1705_01167_b200 import synth  # noqa: E402

g2 = synth.maze_map()
m2 = rl.make_method("cddt", rl.OccupancyGrid.from_array(g2), rl.RangeMethodConfig(500.0, 120))
x, y, t = synth.free_pose(g2, 10, seed=5)
px, py, pt = synth.particles(x, y, t, 2500, 10.0, 0.1, seed=9)
scan = torch.from_numpy(synth.scan(g2, x, y, t, 61, 4.71238898038469, 500.0, 8.0, 0.05, seed=13)).cuda()
beam = rl.BeamModelParams(sigma_hit=8.0, z_max=500.0)
table = torch.from_numpy(rl.beam_table(beam, 501, 1.0)).cuda()
parts = {k: torch.from_numpy(v).cuda() for k, v in dict(x=px, y=py, theta=pt, weight=np.zeros_like(px)).items()}
spec = rl.ScanSpec(61, 4.71238898038469)
f = lambda: rl.sensor_update(parts, m2, scan, spec, beam, table=table)  # noqa: E731
for _ in range(5):
    f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    f()
e1.record()
torch.cuda.synchronize()
print({"ms_per_sensor_update": e0.elapsed_time(e1) / 200})
