"""Where the config-4 particle-filter update time goes: Mcl.step wall and
event time vs a bare ctypes loop of rl_mcl_step. python scripts/pf_overhead.py"""
import ctypes as C
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_01167_b200 as rl  # noqa: E402
from paper_1705_01167_b200 import _lib, mcl, synth  # noqa: E402

g = synth.maze_map()
x, y, t = synth.free_pose(g, 15, seed=8)
pose, odo = synth.trajectory(g, x, y, t, 200, 1.0, 15.0, seed=4)
method = rl.make_method("cddt", rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(500.0, 120))
beam = rl.BeamModelParams(sigma_hit=8.0, z_max=500.0)
table = torch.from_numpy(rl.beam_table(beam, 501, 1.0)).cuda()
cfg = mcl.MclConfig(particle_count=40_000, beam=beam, seed=5,
                    motion=mcl.MotionNoise(1.0, 0.0, 0.0, 0.02))
f = mcl.Mcl(method, cfg, table=table)
f.init_gaussian(x, y, t, 10.0, 0.1)
scans = [torch.from_numpy(synth.scan(g, *pose[k + 1], 61, 4.71238898038469, 500.0, 8.0, 0.05,
                                     seed=1000 + k)).cuda() for k in range(200)]
for k in range(5):
    f.step(*odo[k], scans[k])
torch.cuda.synchronize()
res = {}
# 1. Mcl.step: events and host wall
ev, wall = [], []
for k in range(5, 105):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    f.step(*odo[k], scans[k])
    wall.append(time.perf_counter() - t0)
    e1.record()
    e1.synchronize()
    ev.append(e0.elapsed_time(e1))
res["step_event_us_p50"] = 1e3 * float(np.median(ev))
res["step_wall_us_p50"] = 1e6 * float(np.median(wall))
# 2. bare rl_mcl_step through ctypes, prebuilt arguments
L = _lib.lib()
est = (C.c_double * 3)()
p = lambda tt: C.c_void_p(tt.data_ptr())  # noqa: E731
args = [f.cddt.handle, p(f.x), p(f.y), p(f.theta), p(f.weight), f.n_local]
tail = [p(f._scan_dev), 61, cfg.scan.fov, C.byref(f._noise), C.byref(f._bp), p(table), 501, 1.0,
        cfg.seed]
stream = _lib.torch_stream(f.dev)
bare = []
for k in range(105, 200):
    t0 = time.perf_counter()
    L.rl_mcl_step(*args, *odo[k], *tail, k, est, stream)
    bare.append(time.perf_counter() - t0)
res["bare_ctypes_wall_us_p50"] = 1e6 * float(np.median(bare))
# 3. ctypes call overhead alone
t0 = time.perf_counter()
for _ in range(1000):
    L.rl_last_error()
res["ctypes_noop_us"] = (time.perf_counter() - t0) * 1e3
print(res)
