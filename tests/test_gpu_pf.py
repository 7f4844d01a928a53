"""GPU parity of the particle-filter stages (proj/src/mcl.cpp:42-56, 122-142,
176-201) against the restatement in oracle/cddt_oracle.c, which uses the same
counter-based Philox noise.

Tolerances: motion uses CUDA vs glibc log/sincos (ulp-level), so poses match
within 1e-12 relative; resampling picks the same particles unless a comb
position sits within rounding of a cumulative-weight boundary (the GPU scan
associates the sum differently), which the random weights here never do;
weights within 1e-5 relative (BASELINE.json north_star)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FOV = 4.71238898038469


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _p(t):
    return t.data_ptr()


def orc_motion(oracle_mod, x, y, t, off, dx, dy, dth, noise, seed, it):
    L = oracle_mod.orc_lib()
    L.orc_motion_update.argtypes = [C.c_void_p] * 3 + [C.c_long, C.c_uint64] + [C.c_double] * 3 + \
        [C.c_void_p, C.c_uint64, C.c_uint64]
    nz = np.array(noise, np.float64)
    L.orc_motion_update(x.ctypes.data, y.ctypes.data, t.ctypes.data, x.size, off, dx, dy, dth,
                        nz.ctypes.data, seed, it)


def orc_resample(oracle_mod, x, y, t, w, seed, it):
    L = oracle_mod.orc_lib()
    L.orc_resample.argtypes = [C.c_void_p] * 4 + [C.c_long] + [C.c_void_p] * 5 + [C.c_uint64] * 2
    n = x.size
    out = [np.empty(n) for _ in range(4)]
    src = np.empty(n, np.int64)
    L.orc_resample(x.ctypes.data, y.ctypes.data, t.ctypes.data, w.ctypes.data, n,
                   *(o.ctypes.data for o in out), src.ctypes.data, seed, it)
    return out, src


def test_motion_update_vs_oracle(rl, oracle_mod):
    import torch
    from paper_1705_01167_b200 import _lib
    rng = np.random.default_rng(1)
    n = 40_000
    x, y = rng.uniform(0, 2000, n), rng.uniform(0, 2000, n)
    t = rng.uniform(0, 2 * np.pi, n)
    noise = (0.12, 1.0, 0.25, 0.008)
    for off, it in ((0, 0), (12345, 7)):
        gx, gy, gt = dev(x), dev(y), dev(t)
        nz = _lib.rl_motion_noise_t(*noise)
        _lib.check(_lib.lib().rl_motion_update(_p(gx), _p(gy), _p(gt), n, off, 1.5, -0.25, 0.05,
                                               C.byref(nz), 99, it, None))
        torch.cuda.synchronize()
        ox, oy, ot = x.copy(), y.copy(), t.copy()
        orc_motion(oracle_mod, ox, oy, ot, off, 1.5, -0.25, 0.05, noise, 99, it)
        np.testing.assert_allclose(gx.cpu().numpy(), ox, rtol=1e-12, atol=1e-9)
        np.testing.assert_allclose(gy.cpu().numpy(), oy, rtol=1e-12, atol=1e-9)
        d = np.abs(gt.cpu().numpy() - ot)
        assert np.all((d < 1e-9) | (np.abs(d - 2 * np.pi) < 1e-9))


def test_resample_vs_oracle_and_multiplicity(rl, oracle_mod):
    import torch
    from paper_1705_01167_b200 import _lib
    rng = np.random.default_rng(5)
    n = 40_000
    x, y, t = rng.uniform(0, 100, n), rng.uniform(0, 100, n), rng.uniform(0, 6, n)
    w = rng.exponential(1.0, n)
    w /= w.sum()
    gx, gy, gt, gw = dev(x), dev(y), dev(t), dev(w)
    out = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(4)]
    _lib.check(_lib.lib().rl_resample_low_variance(_p(gx), _p(gy), _p(gt), _p(gw), n, 0, n,
                                                   *(_p(o) for o in out), 3, 11, None))
    (ox, oy, ot, ow), src = orc_resample(oracle_mod, x, y, t, w, 3, 11)
    got = [o.cpu().numpy() for o in out]
    np.testing.assert_array_equal(got[0], ox)
    np.testing.assert_array_equal(got[1], oy)
    np.testing.assert_array_equal(got[3], ow)
    # proj/tests/test_mcl.cpp:307-354: multiplicity in {floor(nw), ceil(nw)}
    counts = np.bincount(src, minlength=n)
    nw = n * w
    assert np.all((counts >= np.floor(nw) - 1e-9) & (counts <= np.ceil(nw) + 1e-9))
    # a shard resampling slots [10000, 30000) sees the same comb
    part = [torch.empty(20000, dtype=torch.float64, device="cuda") for _ in range(4)]
    _lib.check(_lib.lib().rl_resample_low_variance(_p(gx), _p(gy), _p(gt), _p(gw), n, 10000,
                                                   20000, *(_p(o) for o in part), 3, 11, None))
    np.testing.assert_array_equal(part[0].cpu().numpy(), ox[10000:30000])


def _cfg2(rl, synth, n, seed=9):
    g = synth.maze_map()
    x, y, t = synth.free_pose(g, 10, seed=5)
    px, py, pt = synth.particles(x, y, t, n, 10.0, 0.1, seed=seed)
    scan = synth.scan(g, x, y, t, 61, FOV, 500.0, 8.0, 0.05, seed=13)
    return g, (x, y, t), px, py, pt, scan


def test_mcl_step_vs_oracle(rl, oracle_mod, synth):
    """One full Mcl::step (motion -> table sensor model -> estimate -> resample)
    on config-4 sizes (40k particles, 61 beams, 2000x2000 maze, theta_disc 120)."""
    import torch
    from paper_1705_01167_b200 import mcl
    n = 40_000
    g, pose, px, py, pt, scan = _cfg2(rl, synth, n)
    grid = rl.OccupancyGrid.from_array(g)
    method = rl.make_method("cddt", grid, rl.RangeMethodConfig(500.0, 120))
    beam = rl.BeamModelParams(sigma_hit=8.0, z_max=500.0)
    table = rl.beam_table(beam, 501, 1.0)
    cfg = mcl.MclConfig(particle_count=n, beam=beam, seed=21,
                        motion=mcl.MotionNoise(1.0, 0.0, 0.0, 0.02))
    f = mcl.Mcl(method, cfg, table=dev(table))
    f.set_particles(px, py, pt)
    r = f.step(1.0, 0.0, 0.0, scan)
    got = f.particles()
    # oracle pipeline
    ox, oy, ot = px.copy(), py.copy(), pt.copy()
    orc_motion(oracle_mod, ox, oy, ot, 0, 1.0, 0.0, 0.0, (1.0, 0.0, 0.0, 0.02), 21, 0)
    o = oracle_mod.OracleCddt(g, 120, 500.0)
    lw, w, deg = o.sensor_update(ox, oy, ot, scan, FOV, oracle_mod.beam_params(sigma_hit=8.0,
                                 z_max=500.0), table=table)
    assert r.degenerate == deg
    est = np.zeros(3)
    L = oracle_mod.orc_lib()
    L.orc_estimate.argtypes = [C.c_void_p] * 4 + [C.c_long, C.c_void_p]
    L.orc_estimate(ox.ctypes.data, oy.ctypes.data, ot.ctypes.data, w.ctypes.data, n,
                   est.ctypes.data)
    assert abs(r.estimate.x - est[0]) < 1e-6 and abs(r.estimate.y - est[1]) < 1e-6
    (rx, ry, rt, rw), _ = orc_resample(oracle_mod, ox, oy, ot, w, 21, 0)
    np.testing.assert_allclose(got["x"], rx, rtol=1e-12)
    np.testing.assert_allclose(got["y"], ry, rtol=1e-12)
    np.testing.assert_allclose(got["weight"], 1.0 / n)


def test_mcl_closed_loop_converges(rl, synth):
    """Acceptance-style closed loop (proj/tests/test_acceptance.cpp:350-380):
    the filter tracks a seeded trajectory through the maze."""
    from paper_1705_01167_b200 import mcl
    g = synth.maze_map()
    x, y, t = synth.free_pose(g, 15, seed=8)
    pose, odo = synth.trajectory(g, x, y, t, 60, 2.0, 20.0, seed=4)
    grid = rl.OccupancyGrid.from_array(g)
    method = rl.make_method("cddt", grid, rl.RangeMethodConfig(500.0, 120))
    cfg = mcl.MclConfig(particle_count=4000, seed=3, beam=rl.BeamModelParams(sigma_hit=8.0,
                        z_max=500.0), motion=mcl.MotionNoise(0.1, 0.0, 0.0, 0.01))
    f = mcl.Mcl(method, cfg)
    f.init_gaussian(x, y, t, 6.0, 0.05)
    errs = []
    for k in range(60):
        scan = synth.scan(g, *pose[k + 1], 61, FOV, 500.0, 4.0, 0.0, seed=100 + k)
        r = f.step(*odo[k], scan)
        errs.append(np.hypot(r.estimate.x - pose[k + 1][0], r.estimate.y - pose[k + 1][1]))
    assert np.median(errs[10:]) < 3.0


@pytest.mark.parametrize("n", [40_000, 1000, 3, 70_001])
def test_fused_step_equals_stage_pipeline(rl, synth, n):
    """rl_mcl_step (motion fused into the sensor kernel, one cooperative
    finish kernel) equals the stage entry points of the sharded step run on a
    single rank, bit for bit: the same moment blocks, tile scan and comb."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    from paper_1705_01167_b200 import _lib, mcl
    g, pose, px, py, pt, scan = _cfg2(rl, synth, n)
    method = rl.make_method("cddt", rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(500.0, 120))
    beam = rl.BeamModelParams(sigma_hit=8.0, z_max=500.0)
    table = dev(rl.beam_table(beam, 501, 1.0))
    cfg = mcl.MclConfig(particle_count=n, beam=beam, seed=17,
                        motion=mcl.MotionNoise(1.0, 0.0, 0.0, 0.02))
    fused = mcl.Mcl(method, cfg, table=table)
    staged = mcl.Mcl(method, cfg, table=table)
    staged.stages = mcl.CudaStages(staged, _lib.torch_stream(staged.dev))
    for f in (fused, staged):
        f.set_particles(px, py, pt)
    if not dist.is_initialized():
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        for k in range(4):
            a = fused.step(1.0, 0.0, 0.01, scan)
            b = staged.step(1.0, 0.0, 0.01, scan)
            assert a.degenerate == b.degenerate
            assert abs(a.estimate.x - b.estimate.x) <= 1e-9 * max(1.0, abs(b.estimate.x))
            assert abs(a.estimate.y - b.estimate.y) <= 1e-9 * max(1.0, abs(b.estimate.y))
            pa, pb = fused.particles(), staged.particles()
            for key in ("x", "y", "theta", "weight"):
                np.testing.assert_array_equal(pa[key], pb[key])
    finally:
        dist.destroy_process_group()
