"""Host-side mirror of the reference's range-method interface (rangelib,
/root/reference/proj/include/rangelib/*.hpp), backed by the CUDA library.

Names, argument meaning and error behaviour follow the reference so callers
(and tests) read like the reference's own: ``Cddt(grid, RangeMethodConfig(...))``,
``cast(RayQuery(x, y, theta))``, ``cast_pair``, ``prune``, ``set_occupancy``,
``make_method(MethodKind.pcddt, grid, cfg)``, ``sensor_update(...)``,
``serialize_cddt`` / ``deserialize_cddt``. The batched entry points
(``cast_batch`` and friends) are the new API the GPU path adds.

Every query runs in librl_cddt.so on the device; this module only marshals.
Device arrays are torch CUDA tensors (plumbing); host arrays are numpy.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import (LogicError, ParseError, check, lib, rl_beam_params_t, rl_cddt_info_t,
                   torch_stream)

kTwoPi = 6.283185307179586476925286766559  # raycast.hpp:12

__all__ = [
    "kTwoPi", "OccupancyGrid", "RangeMethodConfig", "RayQuery", "iround", "normalize_angle_2pi",
    "direction_index", "Cddt", "RangeMethod", "CddtMethod", "MethodKind", "make_method",
    "method_kind_from_name", "serialize_cddt", "deserialize_cddt", "BeamModelParams", "ScanSpec",
    "beam_likelihood", "beam_table", "sensor_update", "ParseError", "LogicError",
]


# ---- raycast.hpp:17-40 ----
def iround(v: float) -> int:
    return int(math.ceil(v - 0.5))


def normalize_angle_2pi(t: float) -> float:
    t = math.fmod(t, kTwoPi)
    if t < 0:
        t += kTwoPi
    if t >= kTwoPi:
        t = 0.0
    return t


def direction_index(theta: float, theta_disc: int) -> int:
    i = iround(theta * float(theta_disc) / kTwoPi)
    i = int(math.fmod(i, theta_disc))  # C++ % truncates toward zero
    if i < 0:
        i += theta_disc
    return i


class OccupancyGrid:
    """Row-major binary grid, cell (x, y) at y * width + x (grid.hpp:12-62)."""

    def __init__(self, width: int, height: int, resolution: float = 0.05, cells=None):
        if width <= 0 or height <= 0:
            raise ValueError("grid dimensions must be positive")
        if not resolution > 0.0:
            raise ValueError("resolution must be positive")
        self._w, self._h, self._res = int(width), int(height), float(resolution)
        if cells is None:
            self.cells = np.zeros((self._h, self._w), dtype=np.uint8)
        else:
            a = np.ascontiguousarray(np.asarray(cells, dtype=np.uint8).reshape(self._h, self._w))
            self.cells = (a != 0).astype(np.uint8)

    @classmethod
    def from_array(cls, a, resolution: float = 0.05) -> "OccupancyGrid":
        a = np.asarray(a)
        return cls(a.shape[1], a.shape[0], resolution, a)

    def width(self) -> int:
        return self._w

    def height(self) -> int:
        return self._h

    def resolution(self) -> float:
        return self._res

    def in_bounds(self, x: int, y: int) -> bool:
        return 0 <= x < self._w and 0 <= y < self._h

    def at(self, x: int, y: int) -> bool:
        return bool(self.cells[y, x])

    def set(self, x: int, y: int, occ: bool) -> None:
        self.cells[y, x] = 1 if occ else 0

    def diagonal(self) -> float:
        return math.sqrt(float(self._w) * self._w + float(self._h) * self._h)

    def occupied_count(self) -> int:
        return int(self.cells.sum())

    def raw(self) -> np.ndarray:
        return self.cells.reshape(-1)

    def __eq__(self, o) -> bool:
        return (isinstance(o, OccupancyGrid) and self._w == o._w and self._h == o._h
                and np.array_equal(self.cells, o.cells))


@dataclass
class RangeMethodConfig:
    """raycast.hpp:51-64: theta_disc directions over the full circle, even, >= 4."""
    max_range: float = 0.0
    theta_disc: int = 216

    def validate(self) -> None:
        if self.max_range < 0.0:
            raise ValueError("max_range must be >= 0")
        if self.theta_disc < 4 or self.theta_disc % 2 != 0:
            raise ValueError("theta_disc must be even and >= 4")

    def resolved_max_range(self, grid: OccupancyGrid) -> float:
        return self.max_range if self.max_range > 0.0 else grid.diagonal()


class RayQuery:
    """raycast.hpp:42-49: theta is normalised to [0, 2pi) on construction."""
    __slots__ = ("x", "y", "theta")

    def __init__(self, x: float, y: float, theta: float):
        self.x, self.y, self.theta = float(x), float(y), normalize_angle_2pi(float(theta))


def _ptr(a) -> int | None:
    """Device pointer of a torch tensor (None passes through)."""
    if a is None:
        return None
    return a.data_ptr()


def _cur_stream(t):
    return torch_stream(t.device)


def _check_tensors(device: int, n: int, **arrays) -> None:
    """Every array a batched entry point hands to the C ABI as a raw pointer:
    a contiguous torch CUDA tensor on the structure's device with the dtype the
    entry point expects and exactly n elements (None = optional and absent).
    Raises ValueError instead of letting a kernel read or write out of bounds."""
    import torch
    for name, (t, dtype) in arrays.items():
        if t is None:
            continue
        if not isinstance(t, torch.Tensor):
            raise ValueError(f"{name}: expected a torch CUDA tensor, got {type(t).__name__}")
        if t.device.type != "cuda" or t.device.index != device:
            raise ValueError(f"{name}: tensor on {t.device}, structure on cuda:{device}")
        if t.dtype != dtype:
            raise ValueError(f"{name}: dtype {t.dtype}, expected {dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name}: tensor must be contiguous")
        if t.numel() != n:
            raise ValueError(f"{name}: {t.numel()} elements, expected {n}")


@dataclass
class SliceProjection:
    """cddt.hpp:22-33 (read-only view)."""
    theta: float
    cos_t: float
    sin_t: float
    y_offset: float
    bin_count: int

    def project_x(self, x: float, y: float) -> float:
        return x * self.cos_t + y * self.sin_t

    def project_y(self, x: float, y: float) -> float:
        return -x * self.sin_t + y * self.cos_t + self.y_offset


class ZeroPointBin:
    """Read-only view of one exported bin row (cddt.hpp:45-137)."""

    def __init__(self, values: np.ndarray):
        self._v = values

    def values(self) -> list[float]:
        return [float(v) for v in self._v]

    def array(self) -> np.ndarray:
        return self._v

    def size(self) -> int:
        return int(self._v.size)

    def empty(self) -> bool:
        return self._v.size == 0


class Cddt:
    """GPU-resident CDDT / PCDDT with the reference's Cddt API (cddt.hpp:149-196).

    ``Cddt(grid, cfg)`` builds on ``device``; ``prune()`` turns it into a PCDDT.
    """

    def __init__(self, grid: OccupancyGrid, cfg: RangeMethodConfig | None = None, storage=None,
                 *, device: int = 0, prune: bool = False, _handle=None):
        self._h = None
        if _handle is not None:
            self._h = _handle
        else:
            cfg = cfg or RangeMethodConfig()
            cfg.validate()
            raw = np.ascontiguousarray(grid.raw(), dtype=np.uint8)
            h = C.c_void_p()
            check(lib().rl_cddt_create(raw.ctypes.data, grid.width(), grid.height(),
                                       grid.resolution(), cfg.theta_disc, cfg.max_range,
                                       1 if prune else 0, device, C.byref(h)))
            self._h = h
        self._export = None
        self._refresh()

    @staticmethod
    def build(grid, cfg=None, storage=None, **kw) -> "Cddt":
        return Cddt(grid, cfg, storage, **kw)

    def __del__(self):
        h, self._h = getattr(self, "_h", None), None
        if h is not None and _lib._lib is not None:
            _lib._lib.rl_cddt_destroy(h)

    def close(self) -> None:
        self.__del__()

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def _refresh(self) -> None:
        info = rl_cddt_info_t()
        check(lib().rl_cddt_info(self._h, C.byref(info)))
        self._info = info
        self._export = None

    # ---- accessors (cddt.hpp:186-203) ----
    def info(self) -> rl_cddt_info_t:
        return self._info

    def max_range(self) -> float:
        return self._info.max_range

    def theta_disc(self) -> int:
        return self._info.theta_disc

    def slice_count(self) -> int:
        return self._info.slice_count

    def pruned(self) -> bool:
        return bool(self._info.pruned)

    def zero_point_count(self) -> int:
        return int(self._info.zero_points)

    def memory_bytes(self) -> int:
        return int(self._info.memory_bytes)

    def device_bytes(self) -> int:
        return int(self._info.device_bytes)

    def init_seconds(self) -> float:
        return float(self._info.init_seconds)

    def export(self) -> dict:
        """CSR structure copied to host: slice_row_base, row_off, zp, membership, grid."""
        if self._export is None:
            i = self._info
            srb = np.zeros(i.slice_count + 1, dtype=np.uint32)
            off = np.zeros(i.rows + 1, dtype=np.uint64)
            zp = np.zeros(max(1, i.zero_points), dtype=np.float32)
            mem = np.zeros(i.width * i.height, dtype=np.uint8)
            g = np.zeros(i.width * i.height, dtype=np.uint8)
            check(lib().rl_cddt_export(self._h, srb.ctypes.data, off.ctypes.data, zp.ctypes.data,
                                       mem.ctypes.data, g.ctypes.data))
            self._export = dict(slice_row_base=srb, row_off=off, zp=zp[: i.zero_points],
                                membership=mem.reshape(i.height, i.width),
                                grid=g.reshape(i.height, i.width))
        return self._export

    def grid(self) -> OccupancyGrid:
        e = self.export()
        return OccupancyGrid.from_array(e["grid"], self._info.resolution)

    def membership(self, x: int, y: int) -> bool:
        return bool(self.export()["membership"][y, x])

    def slice(self, s: int) -> SliceProjection:
        K, w, h = self._info.theta_disc, self._info.width, self._info.height
        q4 = 4 * s
        if q4 % K == 0:
            q = (q4 // K) & 3
            c, sn = (1.0, 0.0) if q == 0 else (0.0, 1.0) if q == 1 else (-1.0, 0.0)
        else:
            t = float(s) * kTwoPi / float(K)
            c, sn = math.cos(t), math.sin(t)
        b, cc = -float(w) * sn, float(h) * c
        corners = (0.0, b, cc, b + cc)
        lo, hi = min(corners), max(corners)
        return SliceProjection(float(s) * kTwoPi / float(K), c, sn, -lo, int(math.ceil(hi - lo)) + 1)

    def bin(self, s: int, row: int) -> ZeroPointBin:
        e = self.export()
        g = int(e["slice_row_base"][s]) + row
        a, b = int(e["row_off"][g]), int(e["row_off"][g + 1])
        return ZeroPointBin(e["zp"][a:b])

    # ---- queries (cddt.cpp:207-279) ----
    def cast(self, q: RayQuery) -> float:
        out = C.c_double()
        check(lib().rl_cddt_cast(self._h, q.x, q.y, q.theta, C.byref(out)))
        return out.value

    def cast_pair(self, q: RayQuery) -> tuple[float, float]:
        f, b = C.c_double(), C.c_double()
        check(lib().rl_cddt_cast_pair(self._h, q.x, q.y, q.theta, C.byref(f), C.byref(b)))
        return f.value, b.value

    def cast_batch(self, x, y, theta, out=None, hit=None, stream=None):
        """Batched casts. torch CUDA f32 tensors -> async on the current stream
        (or `stream`); numpy f32 arrays -> pipelined host path, returns numpy."""
        if isinstance(x, np.ndarray):
            x, y, theta = (np.ascontiguousarray(a, dtype=np.float32).reshape(-1)
                           for a in (x, y, theta))
            if not (x.size == y.size == theta.size):
                raise ValueError("x, y and theta must have the same length")
            if hit is not None:
                raise ValueError("hit cells are returned by the device path only")
            res = np.empty_like(x) if out is None else out
            if not (isinstance(res, np.ndarray) and res.dtype == np.float32
                    and res.flags.c_contiguous and res.flags.writeable and res.size == x.size):
                raise ValueError("out must be a writable contiguous float32 array of len(x)")
            check(lib().rl_cddt_cast_batch_host(self._h, x.ctypes.data, y.ctypes.data,
                                                theta.ctypes.data, res.ctypes.data, x.size))
            return res
        import torch
        if out is None:
            out = torch.empty_like(x)
        n = x.numel()
        f32 = torch.float32
        _check_tensors(self._info.device, n, x=(x, f32), y=(y, f32), theta=(theta, f32),
                       out=(out, f32), hit=(hit, torch.int32))
        s = stream if stream is not None else _cur_stream(x)
        check(lib().rl_cddt_cast_batch(self._h, _ptr(x), _ptr(y), _ptr(theta), _ptr(out),
                                       _ptr(hit), n, s))
        return out

    def cast_queries(self, queries, out=None):
        """The per-query loop of run_batches (bench.cpp:86-106) over an [n, 3] float64
        array of RayQuery rows (x, y, theta) in host memory; returns float64 ranges."""
        q = np.ascontiguousarray(queries, dtype=np.float64)
        if q.ndim != 2 or q.shape[1] != 3:
            raise ValueError("queries must be an [n, 3] array of (x, y, theta)")
        res = np.empty(q.shape[0], dtype=np.float64) if out is None else out
        if not (isinstance(res, np.ndarray) and res.dtype == np.float64
                and res.flags.c_contiguous and res.flags.writeable and res.size == q.shape[0]):
            raise ValueError("out must be a writable contiguous float64 array of len(queries)")
        check(lib().rl_cddt_cast_queries_host(self._h, q.ctypes.data, res.ctypes.data,
                                              q.shape[0]))
        return res

    def cast_batch_f64(self, x, y, theta, out=None, hit=None, res_row=None, res_idx=None,
                       stream=None):
        import torch
        if out is None:
            out = torch.empty_like(x)
        n, f64 = x.numel(), torch.float64
        _check_tensors(self._info.device, n, x=(x, f64), y=(y, f64), theta=(theta, f64),
                       out=(out, f64), hit=(hit, torch.int32), res_row=(res_row, torch.int64),
                       res_idx=(res_idx, torch.int32))
        s = stream if stream is not None else _cur_stream(x)
        check(lib().rl_cddt_cast_batch_f64(self._h, _ptr(x), _ptr(y), _ptr(theta), _ptr(out),
                                           _ptr(hit), _ptr(res_row), _ptr(res_idx), n, s))
        return out

    def directional_batch(self, x, y, a, out=None, stream=None):
        import torch
        if out is None:
            out = torch.empty_like(x)
        n, f64 = x.numel(), torch.float64
        _check_tensors(self._info.device, n, x=(x, f64), y=(y, f64), a=(a, torch.int32),
                       out=(out, f64))
        s = stream if stream is not None else _cur_stream(x)
        check(lib().rl_cddt_directional_batch(self._h, _ptr(x), _ptr(y), _ptr(a), _ptr(out),
                                              n, s))
        return out

    def exact_cast_batch(self, x, y, theta=None, cos_t=None, sin_t=None, out=None, stream=None):
        """oracle_cast (raycast.cpp:9-16) on this structure's grid (torch CUDA f64)."""
        import torch
        if out is None:
            out = torch.empty_like(x)
        n, f64 = x.numel(), torch.float64
        if (cos_t is None) != (sin_t is None):
            raise ValueError("cos_t and sin_t are given together or not at all")
        if theta is None and cos_t is None:
            raise ValueError("exact casts need theta or cos_t/sin_t")
        _check_tensors(self._info.device, n, x=(x, f64), y=(y, f64), theta=(theta, f64),
                       cos_t=(cos_t, f64), sin_t=(sin_t, f64), out=(out, f64))
        s = stream if stream is not None else _cur_stream(x)
        check(lib().rl_exact_cast_batch(self._h, _ptr(x), _ptr(y), _ptr(theta), _ptr(cos_t),
                                        _ptr(sin_t), _ptr(out), n, s))
        return out

    def simulate_scans(self, x, y, theta, spec: "ScanSpec", max_range: float,
                       noise_sigma: float = 0.0, seed: int = 0, stream_id: int = 0,
                       cos_t=None, sin_t=None, out=None, stream=None):
        """simulate_scan (mcl.cpp:144-154) for a batch of poses on this grid:
        torch CUDA f64 poses -> [n, beam_count] scans. Noise comes from the
        counter generator (seed, stream_id, pose, beam)."""
        import torch
        n = x.numel()
        if out is None:
            out = torch.empty((n, spec.beam_count), dtype=torch.float64, device=x.device)
        f64, nb = torch.float64, spec.beam_count
        _check_tensors(self._info.device, n, x=(x, f64), y=(y, f64), theta=(theta, f64))
        _check_tensors(self._info.device, n * nb, cos_t=(cos_t, f64), sin_t=(sin_t, f64),
                       out=(out, f64))
        s = stream if stream is not None else _cur_stream(x)
        check(lib().rl_simulate_scans(self._h, _ptr(x), _ptr(y), _ptr(theta), n, spec.beam_count,
                                      spec.fov, float(max_range), float(noise_sigma), seed,
                                      stream_id, _ptr(cos_t), _ptr(sin_t), _ptr(out), s))
        return out

    def lut_build(self, theta_disc: int):
        """lut_build (raycast.cpp:62-87) on the GPU: uint16 [theta_disc, h, w] (torch CUDA)."""
        import torch
        i = self._info
        e = torch.empty((theta_disc, i.height, i.width), dtype=torch.int16, device=f"cuda:{i.device}")
        check(lib().rl_lut_build(self._h, theta_disc, e.data_ptr(), _cur_stream(e)))
        return e

    # ---- structure maintenance ----
    def prune(self) -> None:
        check(lib().rl_cddt_prune(self._h))
        self._refresh()

    def set_occupancy(self, x: int, y: int, occupied: bool) -> None:
        try:
            check(lib().rl_cddt_set_occupancy(self._h, int(x), int(y), 1 if occupied else 0))
        finally:
            self._refresh()

    def set_occupancy_batch(self, xy, occupied) -> None:
        xy = np.ascontiguousarray(xy, dtype=np.int32).reshape(-1, 2)
        occ = np.ascontiguousarray(occupied, dtype=np.uint8).reshape(-1)
        try:
            check(lib().rl_cddt_set_occupancy_batch(self._h, xy.ctypes.data, occ.ctypes.data,
                                                    occ.size))
        finally:
            self._refresh()

    def sync(self) -> None:
        check(lib().rl_cddt_sync(self._h))


def serialize_cddt(c: Cddt) -> bytes:
    """serialize_cddt (cddt.cpp:458-500)."""
    size = C.c_size_t()
    check(lib().rl_cddt_serialize(c.handle, None, 0, C.byref(size)))
    buf = (C.c_uint8 * size.value)()
    check(lib().rl_cddt_serialize(c.handle, buf, size.value, C.byref(size)))
    return bytes(buf)


def deserialize_cddt(data: bytes, device: int = 0) -> Cddt:
    """deserialize_cddt (cddt.cpp:502-579); raises ParseError on corrupt input."""
    buf = (C.c_uint8 * max(1, len(data))).from_buffer_copy(data or b"\0")
    h = C.c_void_p()
    check(lib().rl_cddt_deserialize(buf, len(data), device, C.byref(h)))
    return Cddt(None, _handle=h)


class MethodKind(enum.Enum):
    """methods.hpp:15. Only the CDDT family runs on the GPU path."""
    oracle = "oracle"
    bresenham = "bl"
    ray_march = "rm"
    cddt = "cddt"
    pcddt = "pcddt"
    lut = "lut"


def method_kind_from_name(name: str) -> MethodKind:
    for k in MethodKind:
        if k.value == name:
            return k
    raise ValueError(f"unknown method '{name}' (expected bl, rm, cddt, pcddt, lut or oracle)")


class RangeMethod:
    """methods.hpp:22-50."""

    def name(self) -> str:
        raise NotImplementedError

    def cast(self, q: RayQuery) -> float:
        raise NotImplementedError

    def cast_pair(self, q: RayQuery) -> tuple[float, float]:
        return self.cast(q), self.cast(RayQuery(q.x, q.y, q.theta + kTwoPi / 2.0))

    def supports_paired_cast(self) -> bool:
        return False

    def direction_count(self) -> int:
        return 0

    def memory_bytes(self) -> int:
        raise NotImplementedError

    def max_range(self) -> float:
        return self._max_range

    def init_seconds(self) -> float:
        return self._init_seconds


class CddtMethod(RangeMethod):
    """CddtMethod (methods.cpp:79-97) over the GPU structure."""

    def __init__(self, grid: OccupancyGrid, cfg: RangeMethodConfig, prune: bool, device: int = 0):
        self.cddt = Cddt(grid, cfg, device=device, prune=prune)
        self._max_range = self.cddt.max_range()
        self._init_seconds = self.cddt.init_seconds()

    def name(self) -> str:
        return "pcddt" if self.cddt.pruned() else "cddt"

    def cast(self, q: RayQuery) -> float:
        return self.cddt.cast(q)

    def cast_pair(self, q: RayQuery) -> tuple[float, float]:
        return self.cddt.cast_pair(q)

    def supports_paired_cast(self) -> bool:
        return True

    def direction_count(self) -> int:
        return self.cddt.theta_disc()

    def memory_bytes(self) -> int:
        return self.cddt.memory_bytes()


def make_method(kind: MethodKind | str, grid: OccupancyGrid, cfg: RangeMethodConfig | None = None,
                device: int = 0) -> RangeMethod:
    """make_method (methods.cpp:118-133) for the GPU-backed kinds (cddt, pcddt)."""
    if isinstance(kind, str):
        kind = method_kind_from_name(kind)
    cfg = cfg or RangeMethodConfig()
    if kind in (MethodKind.cddt, MethodKind.pcddt):
        return CddtMethod(grid, cfg, kind is MethodKind.pcddt, device)
    raise NotImplementedError(f"method '{kind.value}' is outside the GPU hot path (DESIGN.md)")


# ---- beam sensor model (mcl.hpp / mcl.cpp) ----
@dataclass
class BeamModelParams:
    """mcl.hpp:32-40."""
    w_hit: float = 0.75
    w_short: float = 0.10
    w_max: float = 0.05
    w_rand: float = 0.10
    sigma_hit: float = 2.0
    lambda_short: float = 0.05
    z_max: float = 0.0

    def c(self) -> rl_beam_params_t:
        return rl_beam_params_t(self.w_hit, self.w_short, self.w_max, self.w_rand, self.sigma_hit,
                                self.lambda_short, self.z_max)


@dataclass
class ScanSpec:
    """mcl.hpp:42-51."""
    beam_count: int = 61
    fov: float = 4.71238898038469

    def beam_offset(self, i: int) -> float:
        if self.beam_count <= 1:
            return 0.0
        return -self.fov / 2.0 + self.fov * float(i) / float(self.beam_count - 1)


def beam_likelihood(p: BeamModelParams, expected: float, measured: float) -> float:
    if not p.z_max > 0.0:
        raise ValueError("beam model z_max must be positive")
    return lib().rl_beam_likelihood(C.byref(p.c()), expected, measured)


def beam_table(p: BeamModelParams, zdim: int, inv_res: float = 1.0) -> np.ndarray:
    """T[m][e] = float(beam_likelihood(e/inv_res, m/inv_res)), e, m in [0, zdim)."""
    t = np.empty((zdim, zdim), dtype=np.float32)
    check(lib().rl_beam_table(C.byref(p.c()), zdim, inv_res, t.ctypes.data))
    return t


def sensor_update(particles, method, scan, spec: ScanSpec, beam: BeamModelParams, table=None,
                  inv_res: float = 1.0, logw=None, degenerate=None):
    """sensor_update (mcl.cpp:58-120) on the GPU.

    particles: dict-like with torch CUDA f64 tensors 'x', 'y', 'theta', 'weight'
    (weights are overwritten, as the reference overwrites Particle::weight).
    scan: torch CUDA f64 [beam_count]. table: optional torch CUDA f32 [zdim, zdim].
    Returns False when the weights were degenerate and reset to uniform (this
    waits for the device). With `degenerate` (a torch CUDA int32 [1] tensor) the
    update is only queued on the current stream (rl_sensor_update_async): the
    flag lands in that tensor (1 = degenerate) and the call returns None.
    """
    cddt = method.cddt if isinstance(method, CddtMethod) else method
    if scan.numel() != spec.beam_count:
        raise ValueError("scan length does not match beam count")
    bp = beam
    if not bp.z_max > 0.0:
        bp = BeamModelParams(**{**bp.__dict__, "z_max": cddt.max_range()})
    x, y, t, w = particles["x"], particles["y"], particles["theta"], particles["weight"]
    zdim = 0 if table is None else int(table.shape[0])
    import torch
    dev, n, f64 = cddt.info().device, x.numel(), torch.float64
    _check_tensors(dev, n, x=(x, f64), y=(y, f64), theta=(t, f64), weight=(w, f64),
                   logw=(logw, f64))
    _check_tensors(dev, spec.beam_count, scan=(scan, f64))
    if table is not None:
        if table.dim() != 2 or table.shape[0] != table.shape[1]:
            raise ValueError("table must be square [zdim, zdim]")
        _check_tensors(dev, zdim * zdim, table=(table, torch.float32))
    if degenerate is not None:
        _check_tensors(dev, 1, degenerate=(degenerate, torch.int32))
        check(lib().rl_sensor_update_async(
            cddt.handle, _ptr(x), _ptr(y), _ptr(t), n, _ptr(scan), spec.beam_count, spec.fov,
            C.byref(bp.c()), _ptr(table), zdim, inv_res, _ptr(logw), _ptr(w), _ptr(degenerate),
            _cur_stream(x)))
        return None
    st = check(lib().rl_sensor_update(
        cddt.handle, _ptr(x), _ptr(y), _ptr(t), n, _ptr(scan), spec.beam_count, spec.fov,
        C.byref(bp.c()), _ptr(table), zdim, inv_res, _ptr(logw), _ptr(w), _cur_stream(x)))
    return st != _lib.RL_EDEGENERATE
