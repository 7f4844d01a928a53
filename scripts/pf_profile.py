"""Workload driver for profiling the sensor model and the particle-filter step
(ncu launch lists / full captures): config-4 Mcl steps (40k particles x 61
beams) then config-2 sensor updates (2,500 x 61), both through the public API.

    python scripts/pf_profile.py [steps4] [updates2]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_01167_b200 as rl  # noqa: E402
from paper_1705_01167_b200 import mcl, synth  # noqa: E402

FOV = 4.71238898038469
steps4 = int(sys.argv[1]) if len(sys.argv) > 1 else 20
upd2 = int(sys.argv[2]) if len(sys.argv) > 2 else 20
g = synth.maze_map()
method = rl.make_method("cddt", rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(500.0, 120))
beam = rl.BeamModelParams(sigma_hit=8.0, z_max=500.0)
table = torch.from_numpy(rl.beam_table(beam, 501, 1.0)).cuda()
# config 4
x, y, t = synth.free_pose(g, 15, seed=8)
pose, odo = synth.trajectory(g, x, y, t, steps4, 1.0, 15.0, seed=4)
cfg = mcl.MclConfig(particle_count=40_000, beam=beam, seed=5,
                    motion=mcl.MotionNoise(1.0, 0.0, 0.0, 0.02))
f = mcl.Mcl(method, cfg, table=table)
f.init_gaussian(x, y, t, 10.0, 0.1)
scans = [torch.from_numpy(synth.scan(g, *pose[k + 1], 61, FOV, 500.0, 8.0, 0.05,
                                     seed=1000 + k)).cuda() for k in range(steps4)]
for k in range(steps4):
    f.step(*odo[k], scans[k])
torch.cuda.synchronize()
# config 2
x, y, t = synth.free_pose(g, 10, seed=5)
px, py, pt = synth.particles(x, y, t, 2500, 10.0, 0.1, seed=9)
scan = torch.from_numpy(synth.scan(g, x, y, t, 61, FOV, 500.0, 8.0, 0.05, seed=13)).cuda()
parts = {k: torch.from_numpy(v).cuda() for k, v in
         dict(x=px, y=py, theta=pt, weight=np.zeros_like(px)).items()}
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(upd2):
    rl.sensor_update(parts, method, scan, rl.ScanSpec(61, FOV), beam, table=table, degenerate=flag)
torch.cuda.synchronize()
print("pf_profile done", f.estimate())
