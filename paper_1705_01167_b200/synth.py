"""Seeded synthetic workloads for the BASELINE.json configs (harness side).

Thin ctypes wrapper over csrc/synth.c; see that file for the generators'
definitions. These produce inputs only: maps, query streams, edit rounds,
particle clouds, scans and trajectories.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

_PATH = Path(__file__).resolve().parent / "libcddt_synth.so"
_lib = None
TWO_PI = 6.283185307179586476925286766559


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not _PATH.exists():
            from .build import build_synth
            build_synth()
        h = C.CDLL(str(_PATH))
        P, u64, i32, d = C.c_void_p, C.c_uint64, C.c_int32, C.c_double
        h.synth_rect_map.argtypes = [P, i32, i32, i32, u64]
        h.synth_maze_map.argtypes = [P, i32, i32, d, u64]
        h.synth_polygon_map.argtypes = [P, i32, i32, d, u64]
        h.synth_free_queries.argtypes = [P, i32, i32, u64, C.c_size_t, C.c_size_t, P, P, P]
        h.synth_block_edits.argtypes = [i32, i32, i32, u64, P, P]
        h.synth_block_edits.restype = C.c_long
        h.synth_exact_cast.argtypes = [P, i32, i32, d, d, d, d]
        h.synth_exact_cast.restype = d
        h.synth_free_pose.argtypes = [P, i32, i32, i32, u64, P, P, P]
        h.synth_particles.argtypes = [d, d, d, d, d, u64, C.c_long, P, P, P]
        h.synth_scan.argtypes = [P, i32, i32, d, d, d, i32, d, d, d, d, u64, P]
        h.synth_trajectory.argtypes = [P, i32, i32, d, d, d, C.c_long, d, d, u64, P, P]
        h.synth_map_fnv1a.argtypes = [P, i32, i32]
        h.synth_map_fnv1a.restype = u64
        _lib = h
    return _lib


_gpu = None


def free_queries_gpu(grid_dev, w: int, h: int, n: int, seed=7, start=0, out=None):
    """Device twin of free_queries (csrc/synth_gpu.cu): identical bits, generated on
    the current CUDA device. grid_dev: torch uint8 CUDA tensor [h, w]."""
    import torch
    global _gpu
    if _gpu is None:
        from .build import SYNTH_GPU, build_synth_gpu
        if not SYNTH_GPU.exists():
            build_synth_gpu()
        _gpu = C.CDLL(str(SYNTH_GPU))
        _gpu.synth_free_queries_gpu.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_uint64,
                                                C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p,
                                                C.c_void_p, C.c_void_p]
    if out is None:
        out = tuple(torch.empty(n, dtype=torch.float32, device=grid_dev.device) for _ in range(3))
    qx, qy, qt = out
    stream = C.c_void_p(torch.cuda.current_stream(grid_dev.device).cuda_stream)
    assert _gpu.synth_free_queries_gpu(grid_dev.data_ptr(), w, h, seed, start, n, qx.data_ptr(),
                                       qy.data_ptr(), qt.data_ptr(), stream) == 0
    return qx, qy, qt


def map_fnv1a(grid) -> int:
    """map_content_id's hash (proj/src/bench.cpp:22-34) of a uint8 [h, w] grid."""
    g = np.ascontiguousarray(grid, dtype=np.uint8)
    return int(lib().synth_map_fnv1a(g.ctypes.data, g.shape[1], g.shape[0]))


def rect_map(w=500, h=500, nrect=40, seed=2) -> np.ndarray:
    """Config 1: border + nrect rectangles (side 5-60 px)."""
    g = np.zeros((h, w), dtype=np.uint8)
    assert lib().synth_rect_map(g.ctypes.data, w, h, nrect, seed) == 0
    return g


def maze_map(w=2000, h=2000, occ=0.10, seed=2) -> np.ndarray:
    """Configs 2/4/5: corridor maze (40-120 px rooms, 2-4 px walls, doors)."""
    g = np.zeros((h, w), dtype=np.uint8)
    assert lib().synth_maze_map(g.ctypes.data, w, h, occ, seed) == 0
    return g


def polygon_map(w=4000, h=4000, occ=0.12, seed=3) -> np.ndarray:
    """Config 3: border + filled convex polygons (3-8 vertices, radius 5-60 px)."""
    g = np.zeros((h, w), dtype=np.uint8)
    assert lib().synth_polygon_map(g.ctypes.data, w, h, occ, seed) == 0
    return g


def free_queries(grid: np.ndarray, n: int, seed=7, start=0, out=None):
    """n f32 (x, y, theta) queries uniform over free space; query i depends
    only on (seed, start + i)."""
    h, w = grid.shape
    g = np.ascontiguousarray(grid, dtype=np.uint8)
    if out is None:
        out = (np.empty(n, np.float32), np.empty(n, np.float32), np.empty(n, np.float32))
    qx, qy, qt = out
    lib().synth_free_queries(g.ctypes.data, w, h, seed, start, n, qx.ctypes.data, qy.ctypes.data,
                             qt.ctypes.data)
    return qx, qy, qt


def block_edits(w, h, nblocks=50, seed=11):
    xy = np.zeros((nblocks * 9, 2), dtype=np.int32)
    occ = np.zeros(nblocks * 9, dtype=np.uint8)
    n = lib().synth_block_edits(w, h, nblocks, seed, xy.ctypes.data, occ.ctypes.data)
    return xy[:n], occ[:n]


def exact_cast(grid, x, y, theta, max_range) -> float:
    h, w = grid.shape
    g = np.ascontiguousarray(grid, dtype=np.uint8)
    return lib().synth_exact_cast(g.ctypes.data, w, h, x, y, theta, max_range)


def free_pose(grid, clearance=10, seed=5):
    h, w = grid.shape
    g = np.ascontiguousarray(grid, dtype=np.uint8)
    x, y, t = C.c_double(), C.c_double(), C.c_double()
    assert lib().synth_free_pose(g.ctypes.data, w, h, clearance, seed, C.byref(x), C.byref(y),
                                 C.byref(t)) == 0
    return x.value, y.value, t.value


def particles(x, y, theta, n, sxy=10.0, sth=0.1, seed=9):
    px, py, pt = (np.empty(n, np.float64) for _ in range(3))
    lib().synth_particles(x, y, theta, sxy, sth, seed, n, px.ctypes.data, py.ctypes.data,
                          pt.ctypes.data)
    return px, py, pt


def scan(grid, x, y, theta, nbeams=61, fov=4.71238898038469, max_range=500.0, sigma=8.0,
         p_out=0.05, seed=13) -> np.ndarray:
    h, w = grid.shape
    g = np.ascontiguousarray(grid, dtype=np.uint8)
    s = np.empty(nbeams, np.float64)
    lib().synth_scan(g.ctypes.data, w, h, x, y, theta, nbeams, fov, max_range, sigma, p_out, seed,
                     s.ctypes.data)
    return s


def trajectory(grid, x, y, theta, n, step=1.0, lookahead=15.0, seed=17):
    h, w = grid.shape
    g = np.ascontiguousarray(grid, dtype=np.uint8)
    pose = np.empty((n + 1, 3), np.float64)
    odo = np.empty((n, 3), np.float64)
    lib().synth_trajectory(g.ctypes.data, w, h, x, y, theta, n, step, lookahead, seed,
                           pose.ctypes.data, odo.ctypes.data)
    return pose, odo
