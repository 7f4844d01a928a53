"""Monte-Carlo localisation on the GPU: the reference's Mcl (proj/include/
rangelib/mcl.hpp:101-127, proj/src/mcl.cpp:156-201) with particles resident in
HBM and every per-particle loop a kernel of librl_cddt.so.

Single GPU: one C-ABI call per step (rl_mcl_step_async). Across GPUs (Mcl(...,
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

from ._lib import check, lib, rl_motion_noise_t, torch_stream
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


class MclStepResult:
    """The result of Mcl::step (mcl.cpp:189-201): the pose estimate after the
    sensor update (Mcl::estimate, mcl.cpp:176-187) and whether the weights were
    degenerate and reset (sensor_update returned false).

    The estimate is computed on the GPU and copied back into pinned host memory
    asynchronously, so a step never waits for the device: reading `estimate`
    or `degenerate` waits for that copy (`ready()` polls it). `seconds` is the
    host time spent issuing the step."""

    def __init__(self, host=None, event=None, seconds: float = 0.0,
                 estimate: PoseEstimate | None = None, degenerate: bool = False):
        self._host, self._event, self.seconds = host, event, seconds
        self._est, self._deg = estimate, degenerate

    def ready(self) -> bool:
        return self._est is not None or self._event is None or self._event.query()

    def _resolve(self) -> None:
        if self._est is None:
            if self._event is not None:
                self._event.synchronize()
            h = self._host.tolist()
            self._est, self._deg = PoseEstimate(h[0], h[1], h[2]), bool(h[3])
            self._host = self._event = None

    @property
    def estimate(self) -> PoseEstimate:
        self._resolve()
        return self._est

    @property
    def degenerate(self) -> bool:
        self._resolve()
        return self._deg


def _p(t):
    return None if t is None else t.data_ptr()


class Mcl:
    """Particle filter over a GPU CDDT. `table` (optional, torch f32 [zdim, zdim]
    on the device) selects the discretised likelihood T[m][e] instead of the
    analytic beam model."""

    _RING = 16  # pinned estimate slots (steps that may be in flight)

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
        # this rank's particles as the rows of one [4, n_local] block {x, y, theta, w}:
        # the block is what the resampling all-gather sends, with no packing copy
        self.pblock = torch.zeros((4, self.n_local), **f64)
        self.x, self.y, self.theta, self.weight = self.pblock.unbind(0)
        self.weight.fill_(1.0 / n)
        self.iteration = 0
        self._last: MclStepResult | None = None
        self._scan_dev = torch.empty(cfg.scan.beam_count, **f64)
        self._bp = self.cfg.beam.c()
        self._noise = cfg.motion.c()
        # {x, y, theta, degenerate} of each step. On a GPU the kernels write it straight into a
        # ring of pinned host slots (device-visible under unified addressing): no copy operation
        # on the stream; a slot is reused only after the step that last wrote it completed.
        if self.dev.type == "cuda":
            self._ring = torch.zeros((self._RING, 4), dtype=torch.float64, pin_memory=True)
            self._ring_users = [None] * self._RING
            self.est_dev = self._ring[0]
        else:
            self.est_dev = torch.zeros(4, **f64)
        # stage buffers of the sharded path
        self.logw = torch.empty(self.n_local, **f64)
        self.gmax = torch.empty(1, **f64)
        self.moments = torch.empty(10, **f64)
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.gathered = torch.empty((self.world * 4, self.n_local), **f64)

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
        """Mcl::estimate after the last step (waits for it)."""
        return self._last.estimate if self._last is not None else PoseEstimate()

    # ---- Mcl::step (mcl.cpp:189-201) ----
    def step(self, odo_dx, odo_dy, odo_dtheta, scan) -> MclStepResult:
        """One filter step, issued without waiting for the device: motion,
        sensor model, normalisation, estimate and resampling are queued on the
        current stream (single GPU: two kernels, rl_mcl_step_async; sharded:
        the stages with NCCL exchanges between them). The returned result
        resolves its estimate when read."""
        import torch
        if len(scan) != self.cfg.scan.beam_count:
            raise ValueError("scan length does not match beam count")  # mcl.cpp:61-62
        t0 = time.perf_counter()
        scan_ptr = None
        if (isinstance(scan, torch.Tensor) and scan.device == self.dev
                and scan.dtype == torch.float64 and scan.is_contiguous()):
            scan_ptr = scan.data_ptr()  # read in place, in stream order
        elif isinstance(scan, torch.Tensor):
            self._scan_dev.copy_(scan, non_blocking=True)
        else:
            # through pinned memory: a pageable host->device copy would wait for the stream
            src = torch.from_numpy(np.ascontiguousarray(scan, np.float64))
            if self.dev.type == "cuda":
                src = src.pin_memory()
            self._scan_dev.copy_(src, non_blocking=True)
        self._scan_ptr = scan_ptr if scan_ptr is not None else self._scan_dev.data_ptr()
        cuda = self.dev.type == "cuda"
        stream = torch_stream(self.dev) if cuda else None
        it = self.iteration
        self.iteration += 1
        if cuda:  # this step's pinned estimate slot
            k = it % self._RING
            prev = self._ring_users[k]
            if prev is not None:
                prev._resolve()  # the step that last wrote the slot is done before it is reused
            self.est_dev = self._ring[k]
        if self.world == 1 and self.stages is None:
            check(lib().rl_mcl_step_async(
                self.cddt.handle, _p(self.x), _p(self.y), _p(self.theta), _p(self.weight),
                self.n_local, odo_dx, odo_dy, odo_dtheta, self._scan_ptr,
                self.cfg.scan.beam_count, self.cfg.scan.fov, C.byref(self._noise),
                C.byref(self._bp), _p(self.table), self.zdim, self.inv_res, self.cfg.seed, it,
                _p(self.est_dev), stream))
        else:
            sharded_step(self, self.stages or CudaStages(self, stream), odo_dx, odo_dy,
                         odo_dtheta, it)
        if cuda:
            ev = torch.cuda.Event()
            ev.record(torch.cuda.current_stream(self.dev))
            r = MclStepResult(self.est_dev, ev, time.perf_counter() - t0)
            self._ring_users[k] = r
        else:
            r = MclStepResult(self.est_dev.clone(), None, time.perf_counter() - t0)
        self._last = r
        return r


class CudaStages:
    """The per-shard stages of a sharded step on this rank's GPU, all on one
    stream with no host synchronisation."""

    def __init__(self, m: "Mcl", stream):
        self.m, self.stream = m, stream

    def sensor(self, dx, dy, dth, it):
        """motion_update fused with the shard's log-weights and their max."""
        m = self.m
        check(lib().rl_pf_shard_sensor(
            m.cddt.handle, _p(m.x), _p(m.y), _p(m.theta), m.n_local, m.offset, dx, dy, dth,
            C.byref(m._noise), m.cfg.seed, it, m._scan_ptr, m.cfg.scan.beam_count,
            m.cfg.scan.fov, C.byref(m._bp), _p(m.table), m.zdim, m.inv_res, _p(m.logw),
            _p(m.gmax), self.stream))

    def weights(self):
        m = self.m
        check(lib().rl_pf_weights(_p(m.logw), _p(m.gmax), _p(m.x), _p(m.y), _p(m.theta),
                                  m.n_local, _p(m.weight), _p(m.moments), self.stream))

    def normalize(self):
        m = self.m
        check(lib().rl_pf_normalize(_p(m.weight), m.n_local, _p(m.moments),
                                    m.cfg.particle_count, _p(m.flag), self.stream))

    def estimate(self):
        m = self.m
        check(lib().rl_pf_estimate(_p(m.moments), _p(m.flag), m.cfg.particle_count,
                                   _p(m.est_dev), self.stream))

    def resample(self, it):
        m = self.m
        check(lib().rl_resample_gathered(
            _p(m.gathered), m.n_local, m.world, m.offset, m.n_local, _p(m.x), _p(m.y),
            _p(m.theta), _p(m.weight), m.cfg.seed, it, self.stream))


def sharded_step(m: "Mcl", stages, dx, dy, dth, it) -> None:
    """One Mcl::step over particle shards: local stages with the two exchanges
    of SURVEY.md §8e between them, everything stream-ordered (no host
    synchronisation; the estimate lands in m.est_dev). `stages` supplies the
    local work (CUDA in production; tests substitute a host implementation to
    check this orchestration under a gloo group)."""
    import torch
    import torch.distributed as dist
    stages.sensor(dx, dy, dth, it)  # motion, log-weights and the local max
    dist.all_reduce(m.gmax, op=dist.ReduceOp.MAX, group=m.group)  # exchange 1a: max log-weight
    stages.weights()  # exp(logw - max) and pose moments
    dist.all_reduce(m.moments, op=dist.ReduceOp.SUM, group=m.group)  # exchange 1b: weight sum
    stages.normalize()
    stages.estimate()
    # exchange 2: resampling gather of the [4, n_local] blocks, rank-concatenated
    # ([world * 4, n_local]); every rank resamples its own output slots from it
    if m.gathered.device.type == "cuda" and dist.get_backend(m.group) == "nccl":
        dist.all_gather_into_tensor(m.gathered, m.pblock, group=m.group)
    elif m.gathered.device.type == "cuda":
        # gloo (functional checks of this orchestration only): no CUDA all-gather,
        # so the blocks go through host memory
        host = torch.empty((m.world * 4, m.n_local), dtype=torch.float64)
        dist.all_gather(list(host.view(m.world, 4, m.n_local).unbind(0)), m.pblock.cpu(),
                        group=m.group)
        m.gathered.copy_(host)
    else:
        dist.all_gather(list(m.gathered.view(m.world, 4, m.n_local).unbind(0)), m.pblock,
                        group=m.group)
    stages.resample(it)


def _estimate_from_moments(m, n, degenerate) -> PoseEstimate:
    """Mcl::estimate (mcl.cpp:176-187) from the weight moments
    {sum e, sum e x, sum e y, sum e cos, sum e sin, n, sum x, sum y, sum cos, sum sin}
    (host form, used by host-side stages; the GPU computes the same in rl_pf_estimate)."""
    if degenerate:
        sx, sy, sc, ss, sw = m[6] / n, m[7] / n, m[8] / n, m[9] / n, m[5] / n
    else:
        sx, sy, sc, ss, sw = m[1] / m[0], m[2] / m[0], m[3] / m[0], m[4] / m[0], 1.0
    if not sw > 0.0:
        sw = 1.0
    return PoseEstimate(sx / sw, sy / sw, normalize_angle_2pi(math.atan2(ss, sc)))


__all__ = ["Mcl", "MclConfig", "MotionNoise", "PoseEstimate", "MclStepResult", "kTwoPi"]
