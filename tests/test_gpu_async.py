"""GPU: the asynchronous and sharded forms of the particle-filter step, and the
host-side guards of the batched entry points.

* the CudaStages sharded step at world size 2 (gloo, both ranks on cuda:0 —
  functional: gloo moves the all-gather through host memory) equals the
  single-rank fused step (rl_mcl_step_async) within 1e-12;
* Mcl.step issues everything without waiting for the device (a step queued
  behind a long-running kernel returns before that kernel ends);
* rl_sensor_update_async / rl_resample_gathered / rl_pf_estimate equal their
  synchronous / plain counterparts bit for bit;
* structure edits wait for casts already queued on other streams;
* the batched wrappers reject views, wrong dtypes, wrong devices and short
  arrays instead of passing raw pointers through;
* scratch memory goes back to the driver when the last handle is destroyed.
"""
import ctypes as C
import gc
import os
import socket
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FOV = 4.71238898038469


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _maze_setup(rl, synth, n, seed=9):
    g = synth.maze_map()
    x, y, t = synth.free_pose(g, 10, seed=5)
    px, py, pt = synth.particles(x, y, t, n, 10.0, 0.1, seed=seed)
    scan = synth.scan(g, x, y, t, 61, FOV, 500.0, 8.0, 0.05, seed=13)
    return g, px, py, pt, scan


def _filter(rl, g, n, table=True, group=None, seed=17):
    from paper_1705_01167_b200 import mcl
    method = rl.make_method("cddt", rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(500.0, 120))
    beam = rl.BeamModelParams(sigma_hit=8.0, z_max=500.0)
    tab = dev(rl.beam_table(beam, 501, 1.0)) if table else None
    cfg = mcl.MclConfig(particle_count=n, beam=beam, seed=seed,
                        motion=mcl.MotionNoise(1.0, 0.0, 0.0, 0.02))
    return mcl.Mcl(method, cfg, table=tab, group=group)


N2 = 20_000
STEPS2 = 4


def _rank(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1705_01167_b200 as rl
        from paper_1705_01167_b200 import synth
        g, px, py, pt, scan = _maze_setup(rl, synth, N2)
        f = _filter(rl, g, N2, group=dist.group.WORLD)
        f.set_particles(px, py, pt)
        sdev = dev(scan)
        ests = []
        for k in range(STEPS2):
            r = f.step(1.0, 0.0, 0.01 * k, sdev)
            ests.append((r.estimate.x, r.estimate.y, r.estimate.theta, r.degenerate))
        full = [torch.empty(4, f.n_local, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(full, f.pblock.cpu())
        if rank == 0:
            q.put((torch.cat(full, dim=1).numpy(), ests))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(900)
def test_sharded_cuda_stages_world2_equal_fused(rl, synth):
    """the sharded CudaStages step (rl_pf_shard_sensor, the
    max/sum all-reduces, rl_pf_weights/normalize/estimate, the all-gather and
    rl_resample_gathered) at world size 2 equals the single-GPU fused step."""
    import torch.multiprocessing as mp
    g, px, py, pt, scan = _maze_setup(rl, synth, N2)
    f = _filter(rl, g, N2)
    f.set_particles(px, py, pt)
    sdev = dev(scan)
    one = []
    for k in range(STEPS2):
        r = f.step(1.0, 0.0, 0.01 * k, sdev)
        one.append((r.estimate.x, r.estimate.y, r.estimate.theta, r.degenerate))
    one_p = f.pblock.cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    procs = [ctx.Process(target=_rank, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    two_p, two = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # per-particle stages are identical; only the association of the
    # normalising sums (per rank, then all-reduced) differs
    np.testing.assert_allclose(two_p, one_p, rtol=1e-12, atol=1e-12)
    for a, b in zip(one, two):
        np.testing.assert_allclose(a[:3], b[:3], rtol=1e-12, atol=1e-12)
        assert a[3] == b[3]


def test_step_issues_without_waiting(rl, synth):
    """Mcl.step never synchronises: queued behind a ~0.5 s kernel it returns
    at once, its result is not ready, and reading it then gives the same
    estimate as the synchronous C-ABI step (rl_mcl_step) on the same input."""
    import torch
    from paper_1705_01167_b200 import _lib
    n = 40_000
    g, px, py, pt, scan = _maze_setup(rl, synth, n)
    f = _filter(rl, g, n)
    f.set_particles(px, py, pt)
    sdev = dev(scan)
    f.step(1.0, 0.0, 0.0, sdev).estimate  # warm-up (allocations, first launches)
    f.set_particles(px, py, pt)
    f.iteration = 0
    torch.cuda.synchronize()
    torch.cuda._sleep(1_000_000_000)  # ~0.5 s of device time on the current stream
    t0 = time.perf_counter()
    r = f.step(1.0, 0.0, 0.0, sdev)
    issued = time.perf_counter() - t0
    assert not r.ready(), "the step waited for the device"
    assert issued < 0.2, issued
    got = (r.estimate.x, r.estimate.y, r.estimate.theta, r.degenerate)
    # the synchronous entry point on the same particles
    g2 = _filter(rl, g, n)
    g2.set_particles(px, py, pt)
    est = (C.c_double * 3)()
    g2._scan_dev.copy_(sdev)
    torch.cuda.synchronize()  # rl_mcl_step(stream=NULL) runs on the handle's own stream
    st = _lib.lib().rl_mcl_step(
        g2.cddt.handle, g2.x.data_ptr(), g2.y.data_ptr(), g2.theta.data_ptr(),
        g2.weight.data_ptr(), n, 1.0, 0.0, 0.0, g2._scan_dev.data_ptr(), 61, FOV,
        C.byref(g2._noise), C.byref(g2._bp), g2.table.data_ptr(), 501, 1.0, 17, 0, est, None)
    assert (st == _lib.RL_EDEGENERATE) == got[3]
    np.testing.assert_allclose(got[:2], list(est)[:2], rtol=1e-15)
    assert abs(got[2] - est[2]) <= 1e-14
    np.testing.assert_array_equal(f.pblock.cpu().numpy(), g2.pblock.cpu().numpy())


@pytest.mark.parametrize("table", [True, False])
def test_sensor_update_async_equals_sync(rl, synth, table):
    import torch
    from paper_1705_01167_b200 import _lib
    n = 2500
    g, px, py, pt, scan = _maze_setup(rl, synth, n)
    m = rl.make_method("cddt", rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(500.0, 120))
    beam = rl.BeamModelParams(sigma_hit=8.0, z_max=500.0)
    tab = dev(rl.beam_table(beam, 501, 1.0)) if table else None
    parts = {k: dev(v) for k, v in dict(x=px, y=py, theta=pt, weight=np.zeros(n)).items()}
    sdev = dev(scan)
    ok = rl.sensor_update(parts, m, sdev, rl.ScanSpec(61, FOV), beam, table=tab)
    w_sync = parts["weight"].clone()
    w2 = torch.zeros(n, dtype=torch.float64, device="cuda")
    lw = torch.zeros(n, dtype=torch.float64, device="cuda")
    flag = torch.full((1,), 7, dtype=torch.int32, device="cuda")
    st = _lib.lib().rl_sensor_update_async(
        m.cddt.handle, parts["x"].data_ptr(), parts["y"].data_ptr(), parts["theta"].data_ptr(), n,
        sdev.data_ptr(), 61, FOV, C.byref(beam.c()), tab.data_ptr() if table else None,
        501 if table else 0, 1.0, lw.data_ptr(), w2.data_ptr(), flag.data_ptr(),
        _lib.torch_stream(w2.device))
    assert st == 0
    torch.cuda.synchronize()
    assert int(flag[0]) == (0 if ok else 1)
    assert torch.equal(w2, w_sync)


def test_resample_gathered_equals_plain(rl):
    """rl_resample_gathered over a [world][4][n_local] all-gather block picks
    the same particles, bit for bit, as rl_resample_low_variance over the
    concatenated arrays, for every rank's output slots."""
    import torch
    from paper_1705_01167_b200 import _lib
    L = _lib.lib()
    world, nl = 3, 7001
    n = world * nl
    rng = np.random.default_rng(3)
    parts = rng.standard_normal((4, n))
    parts[3] = rng.random(n)
    parts[3] /= parts[3].sum()
    plain = dev(parts)
    gathered = dev(parts.reshape(4, world, nl).transpose(1, 0, 2).copy())
    s = _lib.torch_stream(plain.device)
    for r in range(world):
        a = torch.empty((4, nl), dtype=torch.float64, device="cuda")
        b = torch.empty((4, nl), dtype=torch.float64, device="cuda")
        assert L.rl_resample_low_variance(*(plain[k].data_ptr() for k in range(4)), n, r * nl, nl,
                                          *(a[k].data_ptr() for k in range(4)), 5, 9, s) == 0
        assert L.rl_resample_gathered(gathered.data_ptr(), nl, world, r * nl, nl,
                                      *(b[k].data_ptr() for k in range(4)), 5, 9, s) == 0
        torch.cuda.synchronize()
        assert torch.equal(a, b)


def test_pf_estimate_on_device_matches_host_form(rl):
    import torch
    from paper_1705_01167_b200 import _lib, mcl
    mom = torch.tensor([2.5, 10.0, -4.0, 0.3, -1.2, 1000.0, 7.0, 8.0, 9.0, -3.0],
                       dtype=torch.float64, device="cuda")
    for deg in (0, 1):
        flag = torch.tensor([deg], dtype=torch.int32, device="cuda")
        est = torch.zeros(4, dtype=torch.float64, device="cuda")
        assert _lib.lib().rl_pf_estimate(mom.data_ptr(), flag.data_ptr(), 1000, est.data_ptr(),
                                         None) == 0
        e = mcl._estimate_from_moments(mom.cpu().numpy(), 1000, bool(deg))
        got = est.cpu().numpy()
        np.testing.assert_allclose(got[:2], [e.x, e.y], rtol=1e-15)
        assert abs(got[2] - e.theta) <= 1e-14 and got[3] == deg


def test_edits_wait_for_queued_casts(rl, synth):
    """An edit issued right after casts queued on another stream (no
    synchronisation in between) must not change those casts' results."""
    import torch
    g = synth.maze_map()
    grid = rl.OccupancyGrid.from_array(g)
    c = rl.Cddt(grid, rl.RangeMethodConfig(0.0, 108))
    before = rl.Cddt(grid, rl.RangeMethodConfig(0.0, 108))
    qx, qy, qt = (dev(a) for a in synth.free_queries(g, 8_000_000, seed=31))
    want = before.cast_batch(qx, qy, qt)
    torch.cuda.synchronize()
    side = torch.cuda.Stream()
    for rnd in range(3):
        out = torch.empty_like(qx)
        with torch.cuda.stream(side):
            torch.cuda._sleep(200_000_000)  # the casts start ~0.1 s later
            c.cast_batch(qx, qy, qt, out=out)
        xy, occ = synth.block_edits(2000, 2000, 50, seed=700 + rnd)
        c.set_occupancy_batch(xy, occ)  # no synchronisation before the edit
        side.synchronize()
        assert torch.equal(out, want), f"round {rnd}: casts saw a half-edited structure"
        before.set_occupancy_batch(xy, occ)
        want = before.cast_batch(qx, qy, qt)
        torch.cuda.synchronize()


def test_batched_wrappers_validate_arrays(rl, synth):
    import torch
    g = synth.rect_map()
    c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(300.0, 108))
    q = torch.rand((1000, 3), device="cuda") * 400 + 50
    x, y, t = (q[:, k].contiguous() for k in range(3))
    c.cast_batch(x, y, t)
    with pytest.raises(ValueError, match="contiguous"):
        c.cast_batch(q[:, 0], q[:, 1], q[:, 2])  # column views
    with pytest.raises(ValueError, match="dtype"):
        c.cast_batch(x.double(), y, t)
    with pytest.raises(ValueError, match="elements"):
        c.cast_batch(x, y[:500], t)
    with pytest.raises(ValueError, match="elements"):
        c.cast_batch(x, y, t, out=torch.empty(10, device="cuda"))
    with pytest.raises(ValueError, match="tensor on cpu"):
        c.cast_batch(x, y.cpu(), t)
    with pytest.raises(ValueError, match="dtype"):
        c.cast_batch(x, y, t, hit=torch.empty(1000, dtype=torch.int64, device="cuda"))
    with pytest.raises(ValueError, match="dtype"):
        c.cast_batch_f64(x, y, t)
    with pytest.raises(ValueError, match="dtype"):
        c.directional_batch(x.double(), y.double(), torch.zeros(1000, device="cuda"))
    hx, hy, ht = (a.cpu().numpy() for a in (x, y, t))
    with pytest.raises(ValueError, match="float32"):
        c.cast_batch(hx, hy, ht, out=np.empty(1000, np.float64))
    with pytest.raises(ValueError, match="same length"):
        c.cast_batch(hx, hy[:10], ht)


_SCRATCH_PROBE = r"""
import gc, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_1705_01167_b200 as rl
from paper_1705_01167_b200 import synth
torch.cuda.init()
torch.cuda.synchronize()
free0, _ = torch.cuda.mem_get_info()
g = synth.rect_map()
c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(300.0, 108))
n = 32_000_000
qx, qy, qt = (torch.rand(n, device="cuda") * 400 + 50 for _ in range(3))
out = c.cast_batch(qx, qy, qt)
torch.cuda.synchronize()
free1, _ = torch.cuda.mem_get_info()
del c, out, qx, qy, qt
gc.collect()
torch.cuda.synchronize()
torch.cuda.empty_cache()
free2, _ = torch.cuda.mem_get_info()
print("held_mb", (free0 - free1) >> 20, "left_mb", (free0 - free2) >> 20)
"""


def test_scratch_returns_to_driver(rl, tmp_path):
    """The batched cast's stream-ordered scratch (~47 B per query) comes from
    the library's own pool and is trimmed when the last handle goes away (run
    in a fresh process: other tests' handles would keep the pool alive)."""
    import re
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, "-c", _SCRATCH_PROBE, str(root)], capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    m = re.search(r"held_mb (\d+) left_mb (-?\d+)", r.stdout)
    assert m, r.stdout
    held, left = int(m.group(1)), int(m.group(2))
    assert held > 1024, held  # the batch did hold scratch
    assert left < 256, left
