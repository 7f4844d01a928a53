"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes access to
  * the C restatement of the reference's CDDT path (oracle/cddt_oracle.c,
    built into oracle/libcddt_oracle.so), and
  * the unmodified reference itself (oracle/_ref/librangelib_ref.so, compiled
    from /root/reference/proj/src by oracle/Makefile), when it was built.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this package; the product path (paper_1705_01167_b200) never
does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "libcddt_oracle.so"
REF_SO = HERE / "_ref" / "librangelib_ref.so"
REF_ROOT = Path(os.environ.get("RANGELIB_REF_ROOT", "/root/reference/proj"))

_P, _d, _i32, _sz = C.c_void_p, C.c_double, C.c_int32, C.c_size_t


def build(ref: bool = True) -> None:
    """Compile the restatement, and the reference when its sources are present."""
    targets = ["all"]
    if ref and (REF_ROOT / "src" / "cddt.cpp").exists():
        targets.append("ref")
        if (HERE.parent / "paper_1705_01167_b200" / "librl_cddt.so").exists():
            targets.append("dropin")
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


def ref_available() -> bool:
    return REF_SO.exists()


_orc = None
_ref = None


def orc_lib() -> C.CDLL:
    global _orc
    if _orc is None:
        if not ORACLE_SO.exists():
            build(ref=False)
        h = C.CDLL(str(ORACLE_SO))
        h.orc_cddt_create.argtypes = [_P, _i32, _i32, _d, _i32, _d, C.POINTER(_P)]
        h.orc_cddt_destroy.argtypes = [_P]
        h.orc_cddt_load.argtypes = [_P, _i32, _i32, _d, _i32, _d, _P, _P, _P, C.c_int,
                                    C.POINTER(_P)]
        h.orc_cddt_info.argtypes = [_P, _P]
        h.orc_cddt_max_range.argtypes = [_P]
        h.orc_cddt_max_range.restype = _d
        h.orc_cddt_export.argtypes = [_P, _P, _P, _P, _P, _P, _P, _P]
        h.orc_cddt_dirs.argtypes = [_P, _P, _P]
        h.orc_cddt_grid.argtypes = [_P, _P]
        h.orc_cast_batch.argtypes = [_P, _P, _P, _P, _sz, _P, _P, _P, _P, _P, _P, C.c_int]
        h.orc_directional_cast.argtypes = [_P, _d, _d, C.c_int, _P, _P, _P, _P]
        h.orc_directional_cast.restype = _d
        h.orc_cast.argtypes = [_P, _d, _d, _d]
        h.orc_cast.restype = _d
        h.orc_prune.argtypes = [_P, C.c_int]
        h.orc_set_occupancy.argtypes = [_P, C.c_int, C.c_int, C.c_int]
        h.orc_beam_likelihood.argtypes = [_P, _d, _d]
        h.orc_beam_likelihood.restype = _d
        h.orc_beam_table.argtypes = [_P, C.c_int, _d, _P]
        h.orc_sensor_update.argtypes = [_P, _P, _P, _P, C.c_long, _P, C.c_int, _d, _P, _P, C.c_int,
                                        _d, _P, _P, C.c_int]
        h.orc_direction_components.argtypes = [C.c_int, C.c_int, _P, _P]
        h.orc_normalize_angle_2pi.argtypes = [_d]
        h.orc_normalize_angle_2pi.restype = _d
        h.orc_direction_index.argtypes = [_d, C.c_int]
        _orc = h
    return _orc


def ref_lib() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            if (REF_ROOT / "src" / "cddt.cpp").exists():
                build(ref=True)
            else:
                raise FileNotFoundError(f"{REF_SO} not built and reference sources absent")
        h = C.CDLL(str(REF_SO))
        h.ref_cddt_create.argtypes = [_P, _i32, _i32, _d, _i32, _d, _i32, C.POINTER(_P)]
        h.ref_cddt_destroy.argtypes = [_P]
        h.ref_cddt_prune.argtypes = [_P]
        h.ref_cddt_info.argtypes = [_P, _P]
        h.ref_cddt_max_range.argtypes = [_P]
        h.ref_cddt_max_range.restype = _d
        h.ref_cddt_export.argtypes = [_P, _P, _P, _P, _P, _P]
        h.ref_cddt_grid.argtypes = [_P, _P]
        h.ref_cast_batch.argtypes = [_P, _P, _P, _P, _sz, _P, _P, _P, C.c_int]
        h.ref_directional_batch.argtypes = [_P, _P, _P, _P, _sz, _P]
        h.ref_cast_pair_batch.argtypes = [_P, _P, _P, _P, _sz, _P, _P]
        h.ref_set_occupancy.argtypes = [_P, C.c_int, C.c_int, C.c_int]
        h.ref_set_occupancy_timed.argtypes = [_P, _P, _P, _sz, C.POINTER(C.c_int)]
        h.ref_set_occupancy_timed.restype = _d
        h.ref_serialize.argtypes = [_P, _P, _sz]
        h.ref_serialize.restype = _sz
        h.ref_deserialize.argtypes = [_P, _sz, C.POINTER(_P)]
        h.ref_beam_likelihood.argtypes = [_P, _d, _d]
        h.ref_beam_likelihood.restype = _d
        h.ref_sensor_update.argtypes = [_P, _P, _P, _P, C.c_long, _P, C.c_int, _d, _P, _P, C.c_int]
        h.ref_oracle_batch.argtypes = [_P, _P, _P, _P, _sz, _P]
        h.ref_lut_build.argtypes = [_P, C.c_int, _P]
        h.ref_bench.argtypes = [_P, C.c_int, _sz, C.c_uint64, C.c_int, _P, C.c_char_p]
        h.ref_rm_create.argtypes = [_P, _i32, _i32, _d]
        h.ref_rm_create.restype = _P
        h.ref_rm_destroy.argtypes = [_P]
        h.ref_rm_cast_batch.argtypes = [_P, _P, _P, _P, _sz, _P, C.c_int]
        h.ref_cast_batch_cpu1.argtypes = [_P, _P, _P, _P, _sz, _P, _P]
        h.ref_mcl_run.argtypes = [_P, C.c_int, C.c_uint64, _d, _d, _d, _d, _d, _P, _P, C.c_int, _d,
                                  C.c_int, _P, _P, _P, _P]
        _ref = h
    return _ref


def _a(x, dtype):
    return np.ascontiguousarray(x, dtype=dtype)


def _p(a):
    return None if a is None else a.ctypes.data


class _Base:
    """Common export / query surface of the oracle and the reference."""

    def info(self) -> dict:
        out = np.zeros(8, np.int64)
        self._info(self._h, out.ctypes.data)
        keys = ("width", "height", "theta_disc", "slice_count", "rows", "zero_points", "pruned",
                "memory_bytes")
        return dict(zip(keys, (int(v) for v in out)))


class OracleCddt(_Base):
    """C restatement (oracle/cddt_oracle.c)."""

    def __init__(self, grid: np.ndarray, theta_disc: int, max_range: float = 0.0,
                 prune: bool = False, resolution: float = 0.05, threads: int = 0, csr=None):
        """csr: optional dict(row_off, zp, membership, pruned) to load instead of building."""
        L = orc_lib()
        g = _a(grid, np.uint8)
        h, w = g.shape
        self._h = _P()
        if csr is not None:
            off, zp = _a(csr["row_off"], np.uint64), _a(csr["zp"], np.float32)
            mem = _a(csr["membership"], np.uint8)
            st = L.orc_cddt_load(g.ctypes.data, w, h, resolution, theta_disc, max_range,
                                 off.ctypes.data, zp.ctypes.data, mem.ctypes.data,
                                 1 if csr.get("pruned") else 0, C.byref(self._h))
        else:
            st = L.orc_cddt_create(g.ctypes.data, w, h, resolution, theta_disc, max_range,
                                   C.byref(self._h))
        if st:
            raise ValueError(f"oracle create failed ({st})")
        self._info = L.orc_cddt_info
        self.threads = threads or os.cpu_count() or 1
        if prune:
            self.prune()

    def __del__(self):
        if getattr(self, "_h", None) and _orc is not None:
            _orc.orc_cddt_destroy(self._h)
            self._h = None

    def max_range(self) -> float:
        return orc_lib().orc_cddt_max_range(self._h)

    def prune(self) -> None:
        orc_lib().orc_prune(self._h, self.threads)

    def set_occupancy(self, x: int, y: int, occ: bool) -> int:
        return orc_lib().orc_set_occupancy(self._h, x, y, 1 if occ else 0)

    def export(self) -> dict:
        i = self.info()
        srb = np.zeros(i["slice_count"] + 1, np.uint32)
        off = np.zeros(i["rows"] + 1, np.uint64)
        zp = np.zeros(max(1, i["zero_points"]), np.float32)
        mem = np.zeros(i["width"] * i["height"], np.uint8)
        clr = np.zeros_like(mem)
        yoff = np.zeros(i["slice_count"], np.float64)
        nb = np.zeros(i["slice_count"], np.int32)
        orc_lib().orc_cddt_export(self._h, srb.ctypes.data, off.ctypes.data, zp.ctypes.data,
                                  mem.ctypes.data, clr.ctypes.data, yoff.ctypes.data,
                                  nb.ctypes.data)
        return dict(slice_row_base=srb, row_off=off, zp=zp[: i["zero_points"]],
                    membership=mem.reshape(i["height"], i["width"]),
                    clear=clr.reshape(i["height"], i["width"]), y_offset=yoff, bin_count=nb)

    def cast_batch(self, qx, qy, qt, want_f64=True, want_hit=True, want_res=True,
                   want_sectors=False, threads=None):
        qx, qy, qt = _a(qx, np.float32), _a(qy, np.float32), _a(qt, np.float32)
        n = qx.size
        o32 = np.empty(n, np.float32)
        o64 = np.empty(n, np.float64) if want_f64 else None
        hit = np.empty(n, np.int32) if want_hit else None
        rr = np.empty(n, np.int64) if want_res else None
        ri = np.empty(n, np.int32) if want_res else None
        sec = np.empty(n, np.int32) if want_sectors else None
        orc_lib().orc_cast_batch(self._h, qx.ctypes.data, qy.ctypes.data, qt.ctypes.data, n,
                                 o32.ctypes.data, _p(o64), _p(hit), _p(rr), _p(ri), _p(sec),
                                 threads or self.threads)
        return dict(out32=o32, out64=o64, hit=hit, res_row=rr, res_idx=ri, sectors=sec)

    def directional_cast(self, x: float, y: float, a: int) -> float:
        return orc_lib().orc_directional_cast(self._h, x, y, a, None, None, None, None)

    def cast(self, x: float, y: float, theta: float) -> float:
        return orc_lib().orc_cast(self._h, x, y, theta)

    def sensor_update(self, px, py, pt, scan, fov, params, table=None, inv_res=1.0, threads=None):
        px, py, pt, scan = (_a(v, np.float64) for v in (px, py, pt, scan))
        p = _a(params, np.float64)
        n = px.size
        logw, w = np.empty(n), np.empty(n)
        tab = None if table is None else _a(table, np.float32)
        zdim = 0 if tab is None else tab.shape[0]
        deg = orc_lib().orc_sensor_update(self._h, px.ctypes.data, py.ctypes.data, pt.ctypes.data,
                                          n, scan.ctypes.data, scan.size, fov, p.ctypes.data,
                                          _p(tab), zdim, inv_res, logw.ctypes.data, w.ctypes.data,
                                          threads or self.threads)
        return logw, w, bool(deg)


class RefCddt(_Base):
    """The unmodified reference (rangelib::Cddt through oracle/ref_shim.cpp)."""

    def __init__(self, grid=None, theta_disc: int = 216, max_range: float = 0.0,
                 prune: bool = False, resolution: float = 0.05, _handle=None):
        L = ref_lib()
        self._info = L.ref_cddt_info
        if _handle is not None:
            self._h = _handle
            return
        g = _a(grid, np.uint8)
        h, w = g.shape
        self._h = _P()
        st = L.ref_cddt_create(g.ctypes.data, w, h, resolution, theta_disc, max_range,
                               1 if prune else 0, C.byref(self._h))
        if st:
            raise ValueError(f"reference create failed ({st})")

    def __del__(self):
        if getattr(self, "_h", None) and _ref is not None:
            _ref.ref_cddt_destroy(self._h)
            self._h = None

    @classmethod
    def deserialize(cls, data: bytes) -> "RefCddt":
        buf = (C.c_uint8 * len(data)).from_buffer_copy(data)
        h = _P()
        st = ref_lib().ref_deserialize(buf, len(data), C.byref(h))
        if st:
            raise ValueError(f"reference deserialize failed ({st})")
        return cls(_handle=h)

    def serialize(self) -> bytes:
        n = ref_lib().ref_serialize(self._h, None, 0)
        buf = (C.c_uint8 * n)()
        ref_lib().ref_serialize(self._h, buf, n)
        return bytes(buf)

    def max_range(self) -> float:
        return ref_lib().ref_cddt_max_range(self._h)

    def prune(self) -> None:
        ref_lib().ref_cddt_prune(self._h)

    def set_occupancy(self, x: int, y: int, occ: bool) -> int:
        return ref_lib().ref_set_occupancy(self._h, x, y, 1 if occ else 0)

    def set_occupancy_timed(self, xy, occ) -> tuple[int, float]:
        """Cddt::set_occupancy over a batch in order, in C++; (status, seconds)."""
        xy = np.ascontiguousarray(xy, np.int32).reshape(-1, 2)
        occ = np.ascontiguousarray(occ, np.uint8).reshape(-1)
        st = C.c_int(0)
        sec = ref_lib().ref_set_occupancy_timed(self._h, _p(xy), _p(occ), occ.size, C.byref(st))
        return st.value, sec

    def export(self) -> dict:
        i = self.info()
        off = np.zeros(i["rows"] + 1, np.uint64)
        zp = np.zeros(max(1, i["zero_points"]), np.float32)
        mem = np.zeros(i["width"] * i["height"], np.uint8)
        yoff = np.zeros(i["slice_count"], np.float64)
        nb = np.zeros(i["slice_count"], np.int32)
        ref_lib().ref_cddt_export(self._h, off.ctypes.data, zp.ctypes.data, mem.ctypes.data,
                                  yoff.ctypes.data, nb.ctypes.data)
        return dict(row_off=off, zp=zp[: i["zero_points"]],
                    membership=mem.reshape(i["height"], i["width"]), y_offset=yoff, bin_count=nb)

    def cast_batch(self, qx, qy, qt, want_res=True, threads=1):
        qx, qy, qt = _a(qx, np.float32), _a(qy, np.float32), _a(qt, np.float32)
        n = qx.size
        out = np.empty(n, np.float64)
        rr = np.empty(n, np.int64) if want_res else None
        ri = np.empty(n, np.int32) if want_res else None
        ref_lib().ref_cast_batch(self._h, qx.ctypes.data, qy.ctypes.data, qt.ctypes.data, n,
                                 out.ctypes.data, _p(rr), _p(ri), threads)
        return dict(out64=out, res_row=rr, res_idx=ri)

    def directional_batch(self, x, y, a):
        x, y, a = _a(x, np.float64), _a(y, np.float64), _a(a, np.int32)
        out = np.empty(x.size)
        ref_lib().ref_directional_batch(self._h, x.ctypes.data, y.ctypes.data, a.ctypes.data,
                                        x.size, out.ctypes.data)
        return out

    def cast_pair_batch(self, x, y, t):
        x, y, t = _a(x, np.float64), _a(y, np.float64), _a(t, np.float64)
        f, b = np.empty(x.size), np.empty(x.size)
        ref_lib().ref_cast_pair_batch(self._h, x.ctypes.data, y.ctypes.data, t.ctypes.data,
                                      x.size, f.ctypes.data, b.ctypes.data)
        return f, b

    def oracle_batch(self, x, y, t):
        x, y, t = _a(x, np.float64), _a(y, np.float64), _a(t, np.float64)
        out = np.empty(x.size)
        ref_lib().ref_oracle_batch(self._h, x.ctypes.data, y.ctypes.data, t.ctypes.data, x.size,
                                   out.ctypes.data)
        return out

    def bench(self, random_mode: bool, n: int = 0, seed: int = 1, stride: int = 4,
              with_seconds: bool = False):
        """The reference's run_random/grid_benchmark: (queries, checksum, map_id)
        [, total thread-cpu seconds]."""
        out = np.zeros(3)
        mid = C.create_string_buffer(17)
        ref_lib().ref_bench(self._h, 1 if random_mode else 0, n, seed, stride, out.ctypes.data, mid)
        r = (int(out[0]), float(out[1]), mid.value.decode())
        return r + (float(out[2]),) if with_seconds else r

    def cast_batch_cpu1(self, qx, qy, qt):
        """Casts on the calling thread, timed by thread cpu time (the
        reference's benchmark clock): (f64 ranges, cpu seconds)."""
        qx, qy, qt = _a(qx, np.float32), _a(qy, np.float32), _a(qt, np.float32)
        out = np.empty(qx.size)
        sec = np.zeros(1)
        ref_lib().ref_cast_batch_cpu1(self._h, qx.ctypes.data, qy.ctypes.data, qt.ctypes.data,
                                      qx.size, out.ctypes.data, sec.ctypes.data)
        return out, float(sec[0])

    def mcl_run(self, n, seed, pose0, sigma_xy, sigma_th, noise, params, fov, odo, scans):
        """The reference's Mcl (init_gaussian + step per odometry/scan row):
        (per-step MclStepResult.seconds, per-step estimates [k, 3])."""
        odo = _a(odo, np.float64).reshape(-1, 3)
        scans = _a(scans, np.float64)
        it, nb = scans.shape
        nz, p = _a(noise, np.float64), _a(params, np.float64)
        sec, est = np.zeros(it), np.zeros((it, 3))
        st = ref_lib().ref_mcl_run(self._h, n, seed, *pose0, sigma_xy, sigma_th, nz.ctypes.data,
                                   p.ctypes.data, nb, fov, it, odo.ctypes.data, scans.ctypes.data,
                                   sec.ctypes.data, est.ctypes.data)
        if st:
            raise RuntimeError(f"reference Mcl failed ({st})")
        return sec, est

    def lut_build(self, theta_disc):
        i = self.info()
        out = np.empty((theta_disc, i["height"], i["width"]), np.uint16)
        assert ref_lib().ref_lut_build(self._h, theta_disc, out.ctypes.data) == 0
        return out

    def sensor_update(self, px, py, pt, scan, fov, params, paired=False):
        px, py, pt, scan = (_a(v, np.float64) for v in (px, py, pt, scan))
        p = _a(params, np.float64)
        w = np.empty(px.size)
        deg = ref_lib().ref_sensor_update(self._h, px.ctypes.data, py.ctypes.data, pt.ctypes.data,
                                          px.size, scan.ctypes.data, scan.size, fov, p.ctypes.data,
                                          w.ctypes.data, 1 if paired else 0)
        return w, bool(deg)


class RefRayMarch:
    """make_method(ray_march) of the reference (methods.cpp:55-72)."""

    def __init__(self, grid, max_range):
        g = _a(grid, np.uint8)
        h, w = g.shape
        self._h = ref_lib().ref_rm_create(g.ctypes.data, w, h, max_range)

    def __del__(self):
        if getattr(self, "_h", None) and _ref is not None:
            _ref.ref_rm_destroy(self._h)

    def cast_batch(self, qx, qy, qt, threads=1):
        qx, qy, qt = _a(qx, np.float32), _a(qy, np.float32), _a(qt, np.float32)
        out = np.empty(qx.size)
        ref_lib().ref_rm_cast_batch(self._h, qx.ctypes.data, qy.ctypes.data, qt.ctypes.data,
                                    qx.size, out.ctypes.data, threads)
        return out


def beam_params(w_hit=0.75, w_short=0.10, w_max=0.05, w_rand=0.10, sigma_hit=2.0,
                lambda_short=0.05, z_max=0.0) -> np.ndarray:
    return np.array([w_hit, w_short, w_max, w_rand, sigma_hit, lambda_short, z_max], np.float64)
