"""Small workload touching every kernel family of librl_cddt.so, run against
the checked library (-DRL_CHECKED: device bounds assertions, read back through
rl_debug_checks; compute-sanitizer is closed on the GPU pool) built with
-DRL_DEFER_MIN_LOG2=12 so the split cast pipeline (phase 1, near-field kernel,
window passes, continuation queues) runs on small batches;
RL_CDDT_CONT_CAP=1 additionally forces the queue-full path.

    RL_CDDT_LIB=paper_1705_01167_b200/librl_cddt_checked.so python scripts/sanitize_workload.py
"""
import ctypes as C
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_01167_b200 as rl  # noqa: E402
from paper_1705_01167_b200 import _lib, mcl, synth  # noqa: E402

FOV = 4.71238898038469


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


g = synth.maze_map(300, 300, 0.1, 4)
grid = rl.OccupancyGrid.from_array(g)
c = rl.Cddt(grid, rl.RangeMethodConfig(150.0, 24))
p = rl.Cddt(grid, rl.RangeMethodConfig(150.0, 24), prune=True)
# batched casts: split pipeline (>= 2 x 4096 queries in this build), f64 with resolving index
qx, qy, qt = synth.free_queries(g, 20000, seed=3)
for s in (c, p):
    o = s.cast_batch(dev(qx), dev(qy), dev(qt))
    h = s.cast_batch(qx, qy, qt)  # host pipeline
    assert np.array_equal(o.cpu().numpy(), h)
    xd, yd, td = (dev(a.astype(np.float64)) for a in (qx, qy, qt))
    rr = torch.empty(20000, dtype=torch.int64, device="cuda")
    ri = torch.empty(20000, dtype=torch.int32, device="cuda")
    hit = torch.empty(20000, dtype=torch.int32, device="cuda")
    s.cast_batch_f64(xd, yd, td, hit=hit, res_row=rr, res_idx=ri)
    s.directional_batch(xd, yd, (td * 0 + 5).to(torch.int32))
    s.cast(rl.RayQuery(10.5, 20.5, 0.3))
    s.cast_pair(rl.RayQuery(10.5, 20.5, 0.3))
    s.exact_cast_batch(xd[:500], yd[:500], td[:500])
    s.simulate_scans(xd[:50], yd[:50], td[:50], rl.ScanSpec(61, FOV), 150.0, 2.0, seed=1)
c.lut_build(8)
blob = rl.serialize_cddt(p)
q = rl.deserialize_cddt(blob)
assert rl.serialize_cddt(q) == blob
# incremental edits (delta records, sort, warp merge)
for r in range(3):
    xy, occ = synth.block_edits(300, 300, 20, seed=40 + r)
    c.set_occupancy_batch(xy, occ)
c.cast_batch(dev(qx), dev(qy), dev(qt))
# sensor model: small (fused normalisation), large (paired kernel + cooperative normalisation)
beam = rl.BeamModelParams(sigma_hit=8.0, z_max=150.0)
table = dev(rl.beam_table(beam, 151, 1.0))
x0, y0, t0 = synth.free_pose(g, 8, seed=2)
scan = dev(synth.scan(g, x0, y0, t0, 61, FOV, 150.0, 8.0, 0.05, seed=3))
for n in (500, 20000):
    px, py, pt = synth.particles(x0, y0, t0, n, 6.0, 0.1, seed=5)
    parts = {k: dev(v) for k, v in dict(x=px, y=py, theta=pt, weight=np.zeros(n)).items()}
    rl.sensor_update(parts, c, scan, rl.ScanSpec(61, FOV), beam, table=table)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    rl.sensor_update(parts, c, scan, rl.ScanSpec(61, FOV), beam, degenerate=flag)
# particle filter: fused step (cooperative finish), stage entry points
cfg = mcl.MclConfig(particle_count=3000, beam=beam, seed=3,
                    motion=mcl.MotionNoise(1.0, 0.0, 0.0, 0.02))
f = mcl.Mcl(rl.make_method("cddt", grid, rl.RangeMethodConfig(150.0, 24)), cfg, table=table)
f.init_gaussian(x0, y0, t0, 5.0, 0.1)
for k in range(3):
    f.step(1.0, 0.0, 0.01, scan).estimate
L = _lib.lib()
st = _lib.torch_stream(f.dev)
n = 3000
w = torch.rand(n, dtype=torch.float64, device="cuda")
lw = torch.rand(n, dtype=torch.float64, device="cuda")
mx = torch.empty(1, dtype=torch.float64, device="cuda")
mom = torch.empty(10, dtype=torch.float64, device="cuda")
fl = torch.zeros(1, dtype=torch.int32, device="cuda")
est = torch.empty(4, dtype=torch.float64, device="cuda")
L.rl_pf_max(lw.data_ptr(), n, mx.data_ptr(), st)
L.rl_pf_weights(lw.data_ptr(), mx.data_ptr(), f.x.data_ptr(), f.y.data_ptr(), f.theta.data_ptr(),
                n, w.data_ptr(), mom.data_ptr(), st)
L.rl_pf_normalize(w.data_ptr(), n, mom.data_ptr(), n, fl.data_ptr(), st)
L.rl_pf_estimate(mom.data_ptr(), fl.data_ptr(), n, est.data_ptr(), st)
gat = torch.rand((3 * 4, 1000), dtype=torch.float64, device="cuda")
out = torch.empty((4, 1000), dtype=torch.float64, device="cuda")
L.rl_resample_gathered(gat.data_ptr(), 1000, 3, 1000, 1000, *(out[k].data_ptr() for k in range(4)),
                       1, 2, st)
L.rl_pf_shard_sensor(c.handle, f.x.data_ptr(), f.y.data_ptr(), f.theta.data_ptr(), n, 0, 1.0, 0.0,
                     0.0, C.byref(f._noise), 1, 0, scan.data_ptr(), 61, FOV, C.byref(f._bp),
                     table.data_ptr(), 151, 1.0, lw.data_ptr(), mx.data_ptr(), st)
if "--negative" in sys.argv:  # control: an out-of-range direction must trip the assertions
    bad = torch.full((4,), 24, dtype=torch.int32, device="cuda")  # theta_disc is 24
    c.directional_batch(torch.full((4,), 10.5, dtype=torch.float64, device="cuda"),
                        torch.full((4,), 20.5, dtype=torch.float64, device="cuda"), bad)
torch.cuda.synchronize()
nf, code = C.c_uint64(), C.c_uint32()
L.rl_debug_checks(0, C.byref(nf), C.byref(code))
print("sanitize workload done", math.isfinite(f.estimate().x), "device check failures", nf.value,
      "first site", code.value)
assert code.value != 0xFFFFFFFF, "not a checked build"
assert (nf.value > 0) if "--negative" in sys.argv else (nf.value == 0)
