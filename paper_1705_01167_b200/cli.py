"""Command-line front end mirroring the reference CLI (proj/tools/main.cpp:
``rangelib bench|cast|info|mcl-demo|make-map``) for the GPU range methods.

    python -m paper_1705_01167_b200 make-map --kind maze --width 2000 --height 2000 --out maze.pgm
    python -m paper_1705_01167_b200 info  --map maze.pgm --method cddt,pcddt --theta-disc 120
    python -m paper_1705_01167_b200 cast  --map maze.pgm -x 100.5 -y 40.5 --theta 0.3
    python -m paper_1705_01167_b200 bench --map maze.pgm --mode random --queries 10000000 --format jsonl
    python -m paper_1705_01167_b200 mcl-demo --map maze.pgm --particles 40000 --steps 500

Methods: ``cddt`` and ``pcddt``, built and queried on the GPU (reported as
``cddt-gpu`` / ``pcddt-gpu``). Benchmark query streams are the reference's own
(run_random_benchmark / run_grid_benchmark, proj/src/bench.cpp:153-210) and the
report has its fields and formats (bench.hpp:26-47, bench.cpp:235-317); per-query
times come from CUDA events over fixed-size batches instead of a CPU thread clock.
"""
from __future__ import annotations

import argparse
import json
import math
import sys
import time
from pathlib import Path

import numpy as np

from . import rangelib as rl
from . import synth

_GAMMA = np.uint64(0x9E3779B97F4A7C15)


# ---- PGM I/O (load_pgm / save_pgm, proj/src/grid.cpp:49-108) ----
def load_pgm(path: str, threshold: int = 127, resolution: float = 0.05) -> rl.OccupancyGrid:
    data = Path(path).read_bytes()
    if len(data) < 2 or data[0:1] != b"P" or data[1:2] not in (b"2", b"5"):
        raise rl.ParseError("not a P2/P5 pgm (byte 0)")
    binary = data[1:2] == b"5"
    pos = 2

    def token():
        nonlocal pos
        while True:
            while pos < len(data) and data[pos:pos + 1] in b" \t\n\r\v\f":
                pos += 1
            if pos < len(data) and data[pos:pos + 1] == b"#":
                while pos < len(data) and data[pos:pos + 1] != b"\n":
                    pos += 1
                continue
            break
        start = pos
        while pos < len(data) and 48 <= data[pos] <= 57:
            pos += 1
        if start == pos:
            raise rl.ParseError(f"expected a number (byte {start})")
        return int(data[start:pos])

    w, h, maxval = token(), token(), token()
    if w <= 0 or h <= 0:
        raise rl.ParseError(f"bad dimensions (byte {pos})")
    if maxval <= 0 or maxval > 255:
        raise rl.ParseError(f"unsupported maxval (byte {pos})")
    if binary:
        pos += 1  # single whitespace before the raster
        if len(data) - pos < w * h:
            raise rl.ParseError(f"truncated raster (byte {len(data)})")
        px = np.frombuffer(data, np.uint8, w * h, pos).reshape(h, w)
    else:
        px = np.array([token() for _ in range(w * h)], np.int64).reshape(h, w)
    if (px > maxval).any():
        raise rl.ParseError("pixel above maxval")
    return rl.OccupancyGrid.from_array((px <= threshold).astype(np.uint8), resolution)


def save_pgm(grid: rl.OccupancyGrid, path: str) -> None:
    header = f"P5\n{grid.width()} {grid.height()}\n255\n".encode()
    Path(path).write_bytes(header + np.where(grid.cells != 0, 0, 255).astype(np.uint8).tobytes())


def map_content_id(grid: rl.OccupancyGrid) -> str:
    """FNV-1a 64 over dimensions + occupancy (map_content_id, bench.cpp:22-34)."""
    return f"{synth.map_fnv1a(grid.cells):016x}"


def _splitmix_uniforms(seed: int, count: int) -> np.ndarray:
    """SplitMix64(seed).uniform() x count (rng.hpp:9-27), vectorised."""
    k = np.arange(1, count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + k * _GAMMA
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def random_queries(grid: rl.OccupancyGrid, n: int, seed: int):
    """run_random_benchmark's stream (bench.cpp:187-210)."""
    u = _splitmix_uniforms(seed, 3 * n).reshape(n, 3)
    return u[:, 0] * grid.width(), u[:, 1] * grid.height(), u[:, 2] * rl.kTwoPi


def grid_queries(grid: rl.OccupancyGrid, K: int, stride: int):
    """run_grid_benchmark's stream, direction-major (bench.cpp:153-185)."""
    nx = (grid.width() + stride - 1) // stride
    ny = (grid.height() + stride - 1) // stride
    i = np.arange(K * nx * ny, dtype=np.int64)
    ti, r = i // (nx * ny), i % (nx * ny)
    return ((r % nx) * stride + 0.5).astype(np.float64), ((r // nx) * stride + 0.5).astype(
        np.float64), ti.astype(np.float64) * rl.kTwoPi / float(K)


def _method(name: str, grid, cfg, device=0):
    if name not in ("cddt", "pcddt"):
        raise SystemExit(f"method '{name}' is not on the GPU path (cddt, pcddt)")
    return rl.make_method(name, grid, cfg, device=device)


def run_bench(method: rl.CddtMethod, grid, cfg, x, y, t, mode: str, seed: int,
              batch: int = 1 << 20) -> dict:
    """run_batches (bench.cpp:71-150) with CUDA-event-timed device batches."""
    import torch
    n = x.size
    dx, dy, dt = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (x, y, t))
    out = torch.empty_like(dx)
    c = method.cddt
    c.cast_batch_f64(dx[:batch], dy[:batch], dt[:batch], out=out[:batch])  # warm-up batch
    torch.cuda.synchronize()
    records, checksum = [], 0.0
    for s in range(0, n, batch):
        e = min(n, s + batch)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        c.cast_batch_f64(dx[s:e], dy[s:e], dt[s:e], out=out[s:e])
        e1.record()
        e1.synchronize()
        records.append((e - s, e0.elapsed_time(e1) / 1e3))
        checksum += float(np.cumsum(out[s:e].cpu().numpy())[-1])  # in-order sum per batch
    total = sum(r[1] for r in records)
    by = sorted((sec / m, m) for m, sec in records)

    def pct(frac):
        need, cum = frac * n, 0.0
        for v, m in by:
            cum += m
            if cum >= need:
                return v
        return by[-1][0]
    hist = [0.0] * 48
    for v, m in by:
        hist[min(47, max(0, int(math.floor((math.log10(max(v, 1e-300)) + 9.0) * 8.0))))] += m
    return dict(method=method.name() + "-gpu", mode=mode, map_id=map_content_id(grid),
                map_width=grid.width(), map_height=grid.height(), theta_disc=cfg.theta_disc,
                seed=seed, queries=n, batch_size=batch, total_seconds=total, checksum=checksum,
                mean_ns=total / n * 1e9, median_ns=pct(0.5) * 1e9, p25_ns=pct(0.25) * 1e9,
                p75_ns=pct(0.75) * 1e9, p99_ns=pct(0.99) * 1e9, min_ns=by[0][0] * 1e9,
                max_ns=by[-1][0] * 1e9, init_seconds=method.init_seconds(),
                memory_bytes=method.memory_bytes(), speedup_vs_bl=None, histogram=hist)


def emit(reports: list[dict], fmt: str, out=None) -> None:
    """report_emit (bench.cpp:235-317)."""
    out = out or sys.stdout
    if fmt == "jsonl":
        for r in reports:
            out.write(json.dumps(r) + "\n")
    elif fmt == "csv":
        cols = ["method", "mode", "map_id", "map_width", "map_height", "theta_disc", "seed",
                "queries", "batch_size", "total_seconds", "checksum", "mean_ns", "median_ns",
                "p25_ns", "p75_ns", "p99_ns", "min_ns", "max_ns", "init_seconds", "memory_bytes",
                "speedup_vs_bl", "histogram"]
        out.write(",".join(cols) + "\n")
        for r in reports:
            row = [("" if r[k] is None else "|".join(str(int(round(v))) for v in r[k])
                    if k == "histogram" else ("" if r[k] is None else str(r[k]))) for k in cols]
            out.write(",".join(row) + "\n")
    else:
        out.write(f"{'method':<10}{'queries':>12}{'mean(ns)':>12}{'median(ns)':>12}"
                  f"{'p99(ns)':>12}{'init(s)':>12}{'mem(MB)':>12}{'checksum':>18}\n")
        for r in reports:
            out.write(f"{r['method']:<10}{r['queries']:>12}{r['mean_ns']:>12.3f}"
                      f"{r['median_ns']:>12.3f}{r['p99_ns']:>12.3f}{r['init_seconds']:>12.4f}"
                      f"{r['memory_bytes'] / 2**20:>12.2f}{r['checksum']:>18.1f}\n")


def mcl_demo(grid, particles: int, beams: int, fov_deg: float, theta_disc: int, steps: int,
             seed: int, out_csv: str | None) -> dict:
    """Closed-loop localisation on the GPU filter, after run_loop_demo
    (proj/src/demo.cpp:37-118): a circle of radius 0.32 min(w, h) about the
    centre at ~1.5 px per step, noisy odometry and scans, reset to the truth
    when the estimate drifts beyond 20 px."""
    from . import mcl
    cfg = rl.RangeMethodConfig(0.0, theta_disc)
    method = rl.make_method("cddt", grid, cfg)
    g = grid.cells
    step_px, scan_sigma, odo_t, odo_r, reset_px = 1.5, 6.0, 1.5, 0.04, 20.0
    fc = mcl.MclConfig(particle_count=particles, scan=rl.ScanSpec(beams, fov_deg * rl.kTwoPi / 360),
                       beam=rl.BeamModelParams(sigma_hit=scan_sigma), seed=seed)
    fc.motion = mcl.MotionNoise((1.25 * odo_t + 0.05) / step_px, 0.0, 0.0,
                                (1.25 * odo_r + 0.002) / step_px)
    f = mcl.Mcl(method, fc)
    cx, cy = grid.width() / 2.0, grid.height() / 2.0
    radius = 0.32 * min(grid.width(), grid.height())
    dphi = step_px / radius
    rng = np.random.default_rng(seed)
    phi = 0.0
    pose = (cx + radius, cy, rl.kTwoPi / 4)
    f.init_gaussian(*pose, 2.0, 0.05)
    rows, resets = [], 0
    for k in range(steps):
        phi += dphi
        new = (cx + radius * math.cos(phi), cy + radius * math.sin(phi),
               rl.normalize_angle_2pi(phi + rl.kTwoPi / 4))
        wx, wy = new[0] - pose[0], new[1] - pose[1]
        c, s = math.cos(pose[2]), math.sin(pose[2])
        odo = (wx * c + wy * s + odo_t * rng.standard_normal(),
               -wx * s + wy * c + odo_t * rng.standard_normal(),
               (new[2] - pose[2] + math.pi) % rl.kTwoPi - math.pi + odo_r * rng.standard_normal())
        pose = new
        scan = synth.scan(g, *pose, beams, fc.scan.fov, method.max_range(), scan_sigma, 0.0,
                          seed=seed * 100003 + k)
        r = f.step(*odo, scan)
        err = math.hypot(r.estimate.x - pose[0], r.estimate.y - pose[1])
        reset = err > reset_px
        if reset:
            f.init_gaussian(*pose, 2.0, 0.05)
            resets += k >= 10
        rows.append((k, *pose, r.estimate.x, r.estimate.y, r.estimate.theta, err, r.seconds, reset,
                     r.degenerate))
    if out_csv:
        with open(out_csv, "w") as fh:
            fh.write("step,true_x,true_y,true_theta,est_x,est_y,est_theta,error,seconds,reset,"
                     "degenerate\n")
            for row in rows:
                fh.write(",".join(str(int(v)) if isinstance(v, bool) else str(v) for v in row)
                         + "\n")
    errs = [row[7] for row in rows[10:]] or [row[7] for row in rows]
    mean_s = sum(row[8] for row in rows) / len(rows)
    return dict(method="cddt-gpu", median_error=float(np.median(errs)), resets=resets,
                mean_step_seconds=mean_s, particles_at_40hz=particles * 0.025 / mean_s)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1705_01167_b200",
                                 description="GPU CDDT range queries, benchmarks and localisation")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def map_opts(p):
        p.add_argument("--map", required=True, help="occupancy map (PGM, dark pixels occupied)")
        p.add_argument("--threshold", type=int, default=127)
        p.add_argument("--resolution", type=float, default=0.05)

    b = sub.add_parser("bench", help="time range queries")
    map_opts(b)
    b.add_argument("--method", default="cddt,pcddt")
    b.add_argument("--mode", choices=("grid", "random"), default="random")
    b.add_argument("--queries", type=int, default=1_000_000)
    b.add_argument("--stride", type=int, default=4)
    b.add_argument("--theta-disc", type=int, default=216)
    b.add_argument("--max-range", type=float, default=0.0)
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("--format", choices=("table", "csv", "jsonl"), default="table")
    c = sub.add_parser("cast", help="cast a single ray")
    map_opts(c)
    c.add_argument("--method", default="cddt")
    c.add_argument("-x", type=float, required=True)
    c.add_argument("-y", type=float, required=True)
    c.add_argument("--theta", type=float, required=True)
    c.add_argument("--theta-disc", type=int, default=216)
    c.add_argument("--max-range", type=float, default=0.0)
    i = sub.add_parser("info", help="build time and memory")
    map_opts(i)
    i.add_argument("--method", default="cddt,pcddt")
    i.add_argument("--theta-disc", type=int, default=216)
    i.add_argument("--max-range", type=float, default=0.0)
    d = sub.add_parser("mcl-demo", help="closed-loop localisation demo")
    map_opts(d)
    d.add_argument("--particles", type=int, default=1000)
    d.add_argument("--beams", type=int, default=61)
    d.add_argument("--fov-deg", type=float, default=270.0)
    d.add_argument("--theta-disc", type=int, default=216)
    d.add_argument("--steps", type=int, default=200)
    d.add_argument("--seed", type=int, default=1)
    d.add_argument("--out")
    m = sub.add_parser("make-map", help="write a seeded synthetic PGM map")
    m.add_argument("--kind", choices=("rects", "maze", "polygons", "random"), default="maze")
    m.add_argument("--width", type=int, default=500)
    m.add_argument("--height", type=int, default=500)
    m.add_argument("--density", type=float, default=0.05)
    m.add_argument("--seed", type=int, default=1)
    m.add_argument("--out", required=True)
    a = ap.parse_args(argv)

    if a.cmd == "make-map":
        w, h = a.width, a.height
        if a.kind == "rects":
            cells = synth.rect_map(w, h, 40, seed=a.seed)
        elif a.kind == "maze":
            cells = synth.maze_map(w, h, 0.10, seed=a.seed)
        elif a.kind == "polygons":
            cells = synth.polygon_map(w, h, 0.12, seed=a.seed)
        else:  # make_random_map (proj/src/synthetic.cpp:84-93)
            cells = (_splitmix_uniforms(a.seed, w * h) < a.density).reshape(h, w).astype(np.uint8)
        save_pgm(rl.OccupancyGrid.from_array(cells), a.out)
        return 0
    grid = load_pgm(a.map, a.threshold, a.resolution)
    if a.cmd == "cast":
        cfg = rl.RangeMethodConfig(a.max_range, a.theta_disc)
        print(_method(a.method, grid, cfg).cast(rl.RayQuery(a.x, a.y, a.theta)))
        return 0
    if a.cmd == "info":
        cfg = rl.RangeMethodConfig(a.max_range, a.theta_disc)
        for name in a.method.split(","):
            meth = _method(name, grid, cfg)
            print(f"{name}-gpu init={meth.init_seconds():.4f}s memory={meth.memory_bytes()}B "
                  f"zero_points={meth.cddt.zero_point_count()} "
                  f"device={meth.cddt.device_bytes()}B")
        return 0
    if a.cmd == "bench":
        cfg = rl.RangeMethodConfig(a.max_range, a.theta_disc)
        if a.mode == "random":
            x, y, t = random_queries(grid, a.queries, a.seed)
        else:
            x, y, t = grid_queries(grid, a.theta_disc, a.stride)
        reports = [run_bench(_method(n, grid, cfg), grid, cfg, x, y, t, a.mode, a.seed)
                   for n in a.method.split(",")]
        emit(reports, a.format)
        return 0
    if a.cmd == "mcl-demo":
        t0 = time.perf_counter()
        res = mcl_demo(grid, a.particles, a.beams, a.fov_deg, a.theta_disc, a.steps, a.seed,
                       a.out)
        res["wall_seconds"] = time.perf_counter() - t0
        print(json.dumps(res))
        return 0
    return 2


if __name__ == "__main__":
    sys.exit(main())
