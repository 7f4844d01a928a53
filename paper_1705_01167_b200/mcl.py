"""Monte-Carlo localisation on the GPU: the reference's Mcl (proj/include/
rangelib/mcl.hpp:101-127, proj/src/mcl.cpp:156-201) with particles resident in
HBM and every per-particle loop a kernel of librl_cddt.so.

Single GPU: one C-ABI call per step (rl_mcl_step). Across GPUs (Mcl(...,
group=<torch.distributed process group>) with world_size > 1): particles are sharded, the map
and CDDT are replicated on every GPU, and the step runs stage by stage with two
exchanges over NCCL — the weight-sum all-reduce (max log-weight, then the
normalising sum and pose moments) and the resampling all-gather of
(x, y, theta, w) so every rank resamples its own output slots from the global
comb. Motion noise is counter-based, so a particle's draws do
not depend on the sharding.
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field

import numpy as np

from ._lib import RL_EDEGENERATE, check, lib, rl_motion_noise_t, torch_stream
from .rangelib import BeamModelParams, CddtMethod, ScanSpec, kTwoPi, normalize_angle_2pi


@dataclass
class MotionNoise:
    """MotionNoise (mcl.hpp:18-27)."""
    trans_per_trans: float = 0.12
    trans_per_rot: float = 1.0
    rot_per_rot: float = 0.25
    rot_per_trans: float = 0.008

    def c(self) -> rl_motion_noise_t:
        return rl_motion_noise_t(self.trans_per_trans, self.trans_per_rot, self.rot_per_rot,
                                 self.rot_per_trans)


@dataclass
class MclConfig:
    """MclConfig (mcl.hpp:93-99)."""
    particle_count: int = 1000
    scan: ScanSpec = field(default_factory=ScanSpec)
    motion: MotionNoise = field(default_factory=MotionNoise)
    beam: BeamModelParams = field(default_factory=BeamModelParams)
    seed: int = 1


@dataclass
class PoseEstimate:
    x: float = 0.0
    y: float = 0.0
    theta: float = 0.0


@dataclass
class MclStepResult:
    estimate: PoseEstimate
    seconds: float = 0.0
    degenerate: bool = False


def _p(t):
    return None if t is None else t.data_ptr()


class Mcl:
    """Particle filter over a GPU CDDT. `table` (optional, torch f32 [zdim, zdim]
    on the device) selects the discretised likelihood T[m][e] instead of the
    analytic beam model."""

    def __init__(self, method, cfg: MclConfig, table=None, inv_res: float = 1.0, group=None,
                 device=None, stages=None):
        import torch
        import torch.distributed as dist
        self.cddt = method.cddt if isinstance(method, CddtMethod) else method
        self.stages = stages
        if cfg.particle_count <= 0:
            raise ValueError("particle filter needs at least one particle")  # mcl.cpp:158-159
        self.cfg = cfg
        if not cfg.beam.z_max > 0.0:
            self.cfg.beam = BeamModelParams(**{**cfg.beam.__dict__, "z_max": self.cddt.max_range()})
        self.table, self.inv_res = table, inv_res
        self.zdim = 0 if table is None else int(table.shape[0])
        self.dev = device if device is not None else torch.device("cuda", self.cddt.info().device)
        # sharded only when given a process group: a process that merely has
        # torch.distributed initialised (e.g. a multi-rank benchmark) keeps a
        # whole filter of its own
        self.world, self.rank = 1, 0
        self.group = group
        if group is not None:
            self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        n = cfg.particle_count
        if n % self.world:
            raise ValueError(f"particle_count {n} must divide evenly over {self.world} ranks")
        self.n_local = n // self.world
        self.offset = self.rank * self.n_local
        f64 = dict(dtype=torch.float64, device=self.dev)
        self.x = torch.zeros(self.n_local, **f64)
        self.y = torch.zeros(self.n_local, **f64)
        self.theta = torch.zeros(self.n_local, **f64)
        self.weight = torch.full((self.n_local,), 1.0 / n, **f64)
        self.iteration = 0
        self._est = PoseEstimate()
        self._scan_dev = torch.empty(cfg.scan.beam_count, **f64)
        self._bp = self.cfg.beam.c()
        self._noise = cfg.motion.c()
        if True:  # stage buffers for the sharded path
            self.logw = torch.empty(self.n_local, **f64)
            self.gmax = torch.empty(1, **f64)
            self.moments = torch.empty(10, **f64)
            self.flag = torch.zeros(1, dtype=torch.int32, device=self.dev)

    # ---- Mcl::init_gaussian (mcl.cpp:165-174), seeded, shard-independent ----
    def init_gaussian(self, x, y, theta, sigma_xy, sigma_theta):
        import torch
        n = self.cfg.particle_count
        rng = np.random.Generator(np.random.Philox(key=self.cfg.seed))
        px = x + max(sigma_xy, 1e-12) * rng.standard_normal(n)
        py = y + max(sigma_xy, 1e-12) * rng.standard_normal(n)
        pt = np.array([normalize_angle_2pi(theta + max(sigma_theta, 1e-12) * v)
                       for v in rng.standard_normal(n)])
        sl = slice(self.offset, self.offset + self.n_local)
        self.x.copy_(torch.from_numpy(px[sl]))
        self.y.copy_(torch.from_numpy(py[sl]))
        self.theta.copy_(torch.from_numpy(pt[sl]))
        self.weight.fill_(1.0 / n)

    def set_particles(self, x, y, theta, weight=None):
        """Load the full particle set (numpy, length particle_count)."""
        import torch
        sl = slice(self.offset, self.offset + self.n_local)
        for dst, src in ((self.x, x), (self.y, y), (self.theta, theta)):
            dst.copy_(torch.from_numpy(np.ascontiguousarray(src, dtype=np.float64)[sl]))
        if weight is None:
            self.weight.fill_(1.0 / self.cfg.particle_count)
        else:
            self.weight.copy_(torch.from_numpy(np.ascontiguousarray(weight, np.float64)[sl]))

    def particles(self) -> dict:
        """This rank's particles as host arrays (mcl.hpp:116)."""
        return {k: getattr(self, k).cpu().numpy() for k in ("x", "y", "theta", "weight")}

    def estimate(self) -> PoseEstimate:
        return self._est

    # ---- Mcl::step (mcl.cpp:189-201) ----
    def step(self, odo_dx, odo_dy, odo_dtheta, scan) -> MclStepResult:
        import torch
        if len(scan) != self.cfg.scan.beam_count:
            raise ValueError("scan length does not match beam count")  # mcl.cpp:61-62
        t0 = time.perf_counter()
        if isinstance(scan, torch.Tensor):
            self._scan_dev.copy_(scan, non_blocking=True)
        else:
            self._scan_dev.copy_(torch.from_numpy(np.ascontiguousarray(scan, np.float64)))
        stream = torch_stream(self.dev) if self.dev.type == "cuda" else None
        it = self.iteration
        self.iteration += 1
        if self.world == 1 and self.stages is None:
            est = (C.c_double * 3)()
            st = check(lib().rl_mcl_step(
                self.cddt.handle, _p(self.x), _p(self.y), _p(self.theta), _p(self.weight),
                self.n_local, odo_dx, odo_dy, odo_dtheta, _p(self._scan_dev),
                self.cfg.scan.beam_count, self.cfg.scan.fov, C.byref(self._noise),
                C.byref(self._bp), _p(self.table), self.zdim, self.inv_res, self.cfg.seed, it,
                est, stream))
            self._est = PoseEstimate(est[0], est[1], est[2])
            degenerate = st == RL_EDEGENERATE
        else:
            degenerate = self._step_sharded(odo_dx, odo_dy, odo_dtheta, it, stream)
        return MclStepResult(self._est, time.perf_counter() - t0, degenerate)

    def _step_sharded(self, dx, dy, dth, it, stream) -> bool:
        return sharded_step(self, self.stages or CudaStages(self, stream), dx, dy, dth, it)


class CudaStages:
    """The per-shard stages of a sharded step, on this rank's GPU."""

    def __init__(self, m: "Mcl", stream):
        self.m, self.stream = m, stream

    def motion(self, dx, dy, dth, it):
        m = self.m
        check(lib().rl_motion_update(_p(m.x), _p(m.y), _p(m.theta), m.n_local, m.offset, dx, dy,
                                     dth, C.byref(m._noise), m.cfg.seed, it, self.stream))

    def logw(self):
        m = self.m
        check(lib().rl_sensor_logw(m.cddt.handle, _p(m.x), _p(m.y), _p(m.theta), m.n_local,
                                   _p(m._scan_dev), m.cfg.scan.beam_count, m.cfg.scan.fov,
                                   C.byref(m._bp), _p(m.table), m.zdim, m.inv_res, _p(m.logw),
                                   self.stream))
        check(lib().rl_pf_max(_p(m.logw), m.n_local, _p(m.gmax), self.stream))

    def weights(self):
        m = self.m
        check(lib().rl_pf_weights(_p(m.logw), _p(m.gmax), _p(m.x), _p(m.y), _p(m.theta),
                                  m.n_local, _p(m.weight), _p(m.moments), self.stream))

    def normalize(self):
        m = self.m
        check(lib().rl_pf_normalize(_p(m.weight), m.n_local, _p(m.moments),
                                    m.cfg.particle_count, _p(m.flag), self.stream))

    def resample(self, allp, it):
        m = self.m
        check(lib().rl_resample_low_variance(
            _p(allp[0]), _p(allp[1]), _p(allp[2]), _p(allp[3]), m.cfg.particle_count, m.offset,
            m.n_local, _p(m.x), _p(m.y), _p(m.theta), _p(m.weight), m.cfg.seed, it, self.stream))


def sharded_step(m: "Mcl", stages, dx, dy, dth, it) -> bool:
    """One Mcl::step over particle shards: local stages with the two exchanges
    of SURVEY.md §8e between them. `stages` supplies the local work (CUDA in
    production; tests substitute a host implementation to check this
    orchestration under a gloo group)."""
    import torch
    import torch.distributed as dist
    n = m.cfg.particle_count
    stages.motion(dx, dy, dth, it)
    stages.logw()  # logw and the local max
    dist.all_reduce(m.gmax, op=dist.ReduceOp.MAX, group=m.group)  # exchange 1a: max log-weight
    stages.weights()  # exp(logw - max) and pose moments
    dist.all_reduce(m.moments, op=dist.ReduceOp.SUM, group=m.group)  # exchange 1b: weight sum
    stages.normalize()
    both = torch.cat([m.moments, m.flag.to(torch.float64)]).cpu().numpy()  # one read-back
    mom, degenerate = both[:10], bool(both[10])
    m._est = _estimate_from_moments(mom, n, degenerate)
    # exchange 2: resampling gather; every rank resamples its own output slots
    mine = torch.stack([m.x, m.y, m.theta, m.weight])
    # rank-concatenated layout (world*4, n_local): accepted by NCCL and gloo
    flat = torch.empty((m.world * 4, m.n_local), dtype=torch.float64, device=m.x.device)
    if flat.device.type == "cuda":
        dist.all_gather_into_tensor(flat, mine, group=m.group)
    else:
        dist.all_gather(list(flat.view(m.world, 4, m.n_local).unbind(0)), mine, group=m.group)
    full = flat.view(m.world, 4, m.n_local)
    allp = full.permute(1, 0, 2).reshape(4, n).contiguous()
    stages.resample(allp, it)
    return degenerate


def _estimate_from_moments(m, n, degenerate) -> PoseEstimate:
    """Mcl::estimate (mcl.cpp:176-187) from the weight moments
    {sum e, sum e x, sum e y, sum e cos, sum e sin, n, sum x, sum y, sum cos, sum sin}."""
    if degenerate:
        sx, sy, sc, ss, sw = m[6] / n, m[7] / n, m[8] / n, m[9] / n, m[5] / n
    else:
        sx, sy, sc, ss, sw = m[1] / m[0], m[2] / m[0], m[3] / m[0], m[4] / m[0], 1.0
    if not sw > 0.0:
        sw = 1.0
    return PoseEstimate(sx / sw, sy / sw, normalize_angle_2pi(math.atan2(ss, sc)))


__all__ = ["Mcl", "MclConfig", "MotionNoise", "PoseEstimate", "MclStepResult", "kTwoPi"]
