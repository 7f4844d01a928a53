"""CPU, world_size 2 (gloo): the sharded particle-filter step (mcl.sharded_step)
gives the same particles and pose estimate as the unsharded run.

The local stages here are a host implementation built on the oracle (counter-
based motion, sensor log-weights, sequential resampling comb); the thing under
test is the orchestration: shard offsets, the max/sum all-reduces, the moment
bookkeeping and the resampling all-gather with per-rank output slots."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

FOV = 4.71238898038469
N = 96
STEPS = 3


class _Method:
    def __init__(self, mr):
        self._mr = mr

    def max_range(self):
        return self._mr


class HostStages:
    def __init__(self, m, orc, scan, params):
        self.m, self.orc, self.scan, self.params = m, orc, scan, params
        import oracle
        self.L = oracle.orc_lib()

    def _np(self, t):
        return t.numpy()

    def sensor(self, dx, dy, dth, it):
        self.motion(dx, dy, dth, it)
        self.logw()

    def motion(self, dx, dy, dth, it):
        import ctypes as C
        m = self.m
        noise = np.array([m.cfg.motion.trans_per_trans, m.cfg.motion.trans_per_rot,
                          m.cfg.motion.rot_per_rot, m.cfg.motion.rot_per_trans])
        x, y, t = self._np(m.x), self._np(m.y), self._np(m.theta)
        self.L.orc_motion_update.argtypes = [C.c_void_p] * 3 + [C.c_long, C.c_uint64] + \
            [C.c_double] * 3 + [C.c_void_p, C.c_uint64, C.c_uint64]
        self.L.orc_motion_update(x.ctypes.data, y.ctypes.data, t.ctypes.data, m.n_local, m.offset,
                                 dx, dy, dth, noise.ctypes.data, m.cfg.seed, it)

    def logw(self):
        m = self.m
        lw, _, _ = self.orc.sensor_update(self._np(m.x), self._np(m.y), self._np(m.theta),
                                          self.scan, FOV, self.params, threads=1)
        m.logw.copy_(torch.from_numpy(lw))
        m.gmax.fill_(float(lw.max()))

    def weights(self):
        m = self.m
        e = torch.exp(m.logw - m.gmax)
        m.weight.copy_(e)
        c, s = torch.cos(m.theta), torch.sin(m.theta)
        m.moments.copy_(torch.stack([e.sum(), (e * m.x).sum(), (e * m.y).sum(), (e * c).sum(),
                                     (e * s).sum(), torch.tensor(float(m.n_local), dtype=torch.float64),
                                     m.x.sum(), m.y.sum(), c.sum(), s.sum()]))

    def normalize(self):
        m = self.m
        s = float(m.moments[0])
        bad = not (s > 0.0) or not np.isfinite(s)
        if bad:
            m.weight.fill_(1.0 / m.cfg.particle_count)
        else:
            m.weight.div_(s)
        m.flag.fill_(1 if bad else 0)

    def estimate(self):
        from paper_1705_01167_b200 import mcl
        m = self.m
        e = mcl._estimate_from_moments(m.moments.numpy(), m.cfg.particle_count, bool(m.flag[0]))
        m.est_dev.copy_(torch.tensor([e.x, e.y, e.theta, float(m.flag[0])], dtype=torch.float64))

    def resample(self, it):
        import ctypes as C
        m = self.m
        n = m.cfg.particle_count
        # the rank-concatenated all-gather block [world * 4, n_local] -> rows x, y, theta, w
        allp = m.gathered.view(m.world, 4, m.n_local).permute(1, 0, 2).reshape(4, n)
        a = [np.ascontiguousarray(allp[k].numpy()) for k in range(4)]
        out = [np.empty(n) for _ in range(4)]
        self.L.orc_resample.argtypes = [C.c_void_p] * 4 + [C.c_long] + [C.c_void_p] * 5 + \
            [C.c_uint64, C.c_uint64]
        self.L.orc_resample(*(v.ctypes.data for v in a), n, *(v.ctypes.data for v in out), None,
                            m.cfg.seed, it)
        sl = slice(m.offset, m.offset + m.n_local)
        for dst, src in zip((m.x, m.y, m.theta, m.weight), out):
            dst.copy_(torch.from_numpy(src[sl]))


def _run(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_1705_01167_b200 import mcl, synth
        g = synth.maze_map(300, 300, 0.1, 4)
        orc = oracle.OracleCddt(g, 24, 120.0, threads=1)
        x, y, t = synth.free_pose(g, 8, seed=2)
        scan = synth.scan(g, x, y, t, 61, FOV, 120.0, 8.0, 0.05, seed=3)
        params = oracle.beam_params(sigma_hit=8.0, z_max=120.0)
        cfg = mcl.MclConfig(particle_count=N, seed=11)
        cfg.motion = mcl.MotionNoise(1.0, 0.0, 0.0, 0.02)
        cfg.beam.z_max = 120.0
        m = mcl.Mcl(_Method(120.0), cfg, device=torch.device("cpu"), stages=None,
                    group=dist.group.WORLD)
        m.stages = HostStages(m, orc, scan, params)
        px, py, pt = synth.particles(x, y, t, N, 6.0, 0.1, seed=5)
        m.set_particles(px, py, pt)
        ests = []
        for _ in range(STEPS):
            r = m.step(1.0, 0.0, 0.01, scan)
            ests.append((r.estimate.x, r.estimate.y, r.estimate.theta, r.degenerate))
        full = [torch.empty(4, m.n_local, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(full, torch.stack([m.x, m.y, m.theta, m.weight]))
        if rank == 0:
            q.put((torch.cat(full, dim=1).numpy(), ests))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _launch(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.timeout(600)
def test_sharded_step_matches_single_rank(oracle_mod):
    one_p, one_e = _launch(1)
    two_p, two_e = _launch(2)
    # motion draws and log-weights are per particle; only the order of the
    # normalising sum differs between 1 and 2 ranks
    np.testing.assert_allclose(two_p, one_p, rtol=1e-12, atol=1e-12)
    for a, b in zip(one_e, two_e):
        np.testing.assert_allclose(a[:3], b[:3], rtol=1e-12, atol=1e-12)
        assert a[3] == b[3]
