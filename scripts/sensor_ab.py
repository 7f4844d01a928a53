"""A/B timing of the sensor model: config 2 (2,500 x 61 sensor updates,
issued back to back, async flag) and config 4 (40k x 61 Mcl steps, issued back
to back), CUDA events. Library variant via RL_CDDT_LIB, paired beams via
RL_SENSOR_PAIRED. Prints one JSON line.

    RL_SENSOR_PAIRED=0 python scripts/sensor_ab.py
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_01167_b200 as rl  # noqa: E402
from paper_1705_01167_b200 import mcl, synth  # noqa: E402

FOV = 4.71238898038469
g = synth.maze_map()
method = rl.make_method("cddt", rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(500.0, 120))
beam = rl.BeamModelParams(sigma_hit=8.0, z_max=500.0)
table = torch.from_numpy(rl.beam_table(beam, 501, 1.0)).cuda()


def timed(fn, reps):
    for _ in range(5):
        fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(reps):
        fn(k)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


x, y, t = synth.free_pose(g, 10, seed=5)
px, py, pt = synth.particles(x, y, t, 2500, 10.0, 0.1, seed=9)
scan = torch.from_numpy(synth.scan(g, x, y, t, 61, FOV, 500.0, 8.0, 0.05, seed=13)).cuda()
parts = {k: torch.from_numpy(v).cuda() for k, v in
         dict(x=px, y=py, theta=pt, weight=np.zeros_like(px)).items()}
flag = torch.zeros(1, dtype=torch.int32, device="cuda")
spec = rl.ScanSpec(61, FOV)
ms2 = timed(lambda k: rl.sensor_update(parts, method, scan, spec, beam, table=table,
                                       degenerate=flag), 400)
w2 = parts["weight"].clone()
iters = 300
x, y, t = synth.free_pose(g, 15, seed=8)
pose, odo = synth.trajectory(g, x, y, t, iters + 5, 1.0, 15.0, seed=4)
cfg = mcl.MclConfig(particle_count=40_000, beam=beam, seed=5,
                    motion=mcl.MotionNoise(1.0, 0.0, 0.0, 0.02))
f = mcl.Mcl(method, cfg, table=table)
f.init_gaussian(x, y, t, 10.0, 0.1)
scans = [torch.from_numpy(synth.scan(g, *pose[k + 1], 61, FOV, 500.0, 8.0, 0.05,
                                     seed=1000 + k)).cuda() for k in range(iters + 5)]
host = []
ms4 = timed(lambda k: host.append(f.step(*odo[k], scans[k]).seconds), iters)
host_us = 1e6 * float(np.mean(host[5:]))
# the same step through the raw C ABI (no Python Mcl bookkeeping), back to back
import ctypes as C  # noqa: E402

from paper_1705_01167_b200 import _lib  # noqa: E402
L = _lib.lib()
st = _lib.torch_stream(f.dev)
est = torch.zeros(4, dtype=torch.float64, device="cuda")
sptr = [s.data_ptr() for s in scans]


def raw(k):
    L.rl_mcl_step_async(f.cddt.handle, f.x.data_ptr(), f.y.data_ptr(), f.theta.data_ptr(),
                        f.weight.data_ptr(), 40_000, *odo[k], sptr[k], 61, FOV, C.byref(f._noise),
                        C.byref(f._bp), table.data_ptr(), 501, 1.0, 5, 10_000 + k, est.data_ptr(),
                        st)


ms4_raw = timed(raw, iters)
lat = []
for k in range(50):  # one step at a time, estimate read back
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    f.step(*odo[k], scans[k]).estimate
    e1.record()
    e1.synchronize()
    lat.append(e0.elapsed_time(e1))
print(json.dumps(dict(lib=os.environ.get("RL_CDDT_LIB", "default"),
                      paired=os.environ.get("RL_SENSOR_PAIRED", "1"),
                      tail=os.environ.get("RL_SENSOR_TAIL_MAX", "default"),
                      paired_small=os.environ.get("RL_SENSOR_PAIRED_SMALL", "default"),
                      cfg2_ms=ms2, cfg4_ms=ms4, cfg4_raw_abi_ms=ms4_raw,
                      cfg4_host_us_per_step=host_us,
                      cfg4_sync_ms_p50=float(np.median(lat)), w2_sum=float(w2.sum()),
                      est=[f.estimate().x, f.estimate().y])))
