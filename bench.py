#!/usr/bin/env python
"""Benchmark: batched PCDDT ray casts on B200 (BASELINE.json metric
"ray casts/sec (batched CDDT queries)"), workload = BASELINE config 3:
4000x4000 seeded convex-polygon map (~12 % occupied), theta_disc 200,
max_range 1000 px, PCDDT pruning on, 100M uniformly random free-space f32
(x, y, theta) queries per GPU per step (weak scaling: every rank casts its own
100M-query slice of the same seeded stream).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one batched cast of the rank's 100M queries. `value` is timed with
CUDA events on the launching stream with the queries already resident in HBM
(1.2 GB of inputs per step, far above the 126 MB L2, so no L2 flush is needed);
`e2e` times the same batch through the host-pointer C-ABI call
(rl_cddt_cast_batch_host) with the H2D copy of the inputs from pinned memory
and the D2H copy of the ranges inside the timed region.

--impl reference times the reference's own CPU implementation (the unmodified
rangelib compiled into oracle/_ref) on the host cores with all threads. Both
arms also time the reference's ray-marching method on a bounded sample of the
same queries (cpu_baseline.ray_march).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "ray casts/sec (batched CDDT queries)"
UNIT = "casts/s"
WORKLOAD = dict(
    workload="BASELINE config 3: 4000x4000 convex-polygon map (~12% occ), theta_disc=200, "
             "max_range=1000 px, PCDDT, 100M free-space f32 queries per GPU per step",
    map="polygon 4000x4000 occ>=0.12 seed=3", theta_disc=200, max_range=1000.0, pruned=True,
    queries_per_gpu_per_step=100_000_000, query_seed=7, l2="inputs 1.2 GB/step > 126 MB L2 "
    "(no flush needed)")


def workload_config(n: int) -> dict:
    """WORKLOAD with the query count actually used (--queries)."""
    if n == WORKLOAD["queries_per_gpu_per_step"]:
        return dict(WORKLOAD)
    return dict(WORKLOAD, queries_per_gpu_per_step=n,
                workload=WORKLOAD["workload"].replace("100M", f"{n / 1e6:g}M"),
                l2=f"inputs {12 * n / 1e9:.2f} GB/step")


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# ---------------------------------------------------------------- clocks
REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")


class ClockSampler:
    """nvidia-smi sampled every 20 ms; summary() covers the samples after mark()."""

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        q = "clocks.sm,clocks.max.sm," + ",".join(f"clocks_event_reasons.{r}" for r in REASONS)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # the timed region starts once samples flow (nvidia-smi takes a moment to start)
            t0 = time.monotonic()
            while not self.rows and time.monotonic() - t0 < 2.0 and self.proc.poll() is None:
                time.sleep(0.01)
            self.skip = len(self.rows)
        except OSError:
            self.proc = None
        return self

    def mark(self):
        """The timed region starts now: earlier samples are not reported."""
        self.skip = len(self.rows)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 2 + len(REASONS):
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        # drop the samples taken before the timed region began (keep one if nothing else)
        rows = self.rows[getattr(self, "skip", 0):] or self.rows[-1:]
        self.rows = rows
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({REASONS[i] for r in self.rows for i in range(len(REASONS))
                          if r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------- helpers
def measured_hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except (KeyError, ValueError):
            pass
    return 6650.0, "fallback"


def profile_traffic():
    """dram bytes per query of the cast kernel from the committed ncu capture."""
    p = ROOT / "profiles" / "traffic.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except ValueError:
            return None
    return None


def make_workload(n_queries: int, rank: int, on_gpu: bool = True):
    """The config-3 map and this rank's query slice in pinned host memory.
    On a GPU the queries come from the device twin of the generator (bit-identical
    to synth.free_queries, tests/test_gpu_synth.py) — seconds of host time per
    rank otherwise."""
    import numpy as np
    import torch

    from paper_1705_01167_b200 import synth
    g = synth.polygon_map(4000, 4000, 0.12, seed=3)
    pin = torch.cuda.is_available()  # the reference arm also runs on a host without a GPU
    qx, qy, qt = (torch.empty(n_queries, dtype=torch.float32, pin_memory=pin) for _ in range(3))
    if on_gpu and torch.cuda.is_available():
        gd = torch.from_numpy(g).cuda()
        dq = synth.free_queries_gpu(gd, 4000, 4000, n_queries, seed=7, start=rank * n_queries)
        for h, d in zip((qx, qy, qt), dq):
            h.copy_(d)
        del dq, gd
        torch.cuda.synchronize()
    else:
        synth.free_queries(g, n_queries, seed=7, start=rank * n_queries,
                           out=(qx.numpy(), qy.numpy(), qt.numpy()))
    return g, qx, qy, qt, np


REF_PCDDT = ROOT / "oracle" / "_ref" / "cfg3_pcddt.rlc"


def reference_structure(g):
    """The config-3 PCDDT as the unmodified reference built it
    (scripts/make_ref_pcddt.py: Cddt::Cddt + Cddt::prune, ~12 min
    single-threaded), loaded through the reference's own deserialize_cddt
    (cddt.cpp:502-579); its sha256 is committed in oracle/cfg3_pcddt.sha256.
    Returns (handle, snapshot bytes, description, same_config). Without the
    snapshot the reference builds an unpruned CDDT (its prune is outside any
    run budget) and same_config is False."""
    import hashlib

    import oracle
    oracle.build(ref=True)
    if not oracle.ref_available():
        raise RuntimeError("oracle/_ref/librangelib_ref.so not built")
    want = (ROOT / "oracle" / "cfg3_pcddt.sha256").read_text().split()[0]
    if REF_PCDDT.exists():
        blob = REF_PCDDT.read_bytes()
        if hashlib.sha256(blob).hexdigest() != want:
            raise RuntimeError(f"{REF_PCDDT} does not match oracle/cfg3_pcddt.sha256")
        return (oracle.RefCddt.deserialize(blob), blob,
                "the reference-built PCDDT (scripts/make_ref_pcddt.py) loaded via its own "
                "deserialize_cddt", True)
    return (oracle.RefCddt(g, 200, 1000.0, prune=False), None,
            "a reference-built unpruned CDDT (oracle/_ref/cfg3_pcddt.rlc absent: the reference's "
            "single-threaded prune of this map takes ~12 min)", False)


def reference_cpu(ref, qx, qy, qt, sample: int, threads: int, sample1: int):
    """Time the unmodified reference's Cddt::cast on `sample` queries with all
    host threads (wall clock; a std::thread partition over the const cast, safe
    per SPEC.md:341) and on `sample1` queries on one thread, timed by thread cpu
    time as the reference's own benchmark does (proj/src/bench.cpp:52-121)."""
    xs, ys, ts = qx[:sample], qy[:sample], qt[:sample]
    ref.cast_batch(xs[:10000], ys[:10000], ts[:10000], want_res=False, threads=threads)
    t0 = time.perf_counter()
    r = ref.cast_batch(xs, ys, ts, want_res=False, threads=threads)
    dt = time.perf_counter() - t0
    _, sec1 = ref.cast_batch_cpu1(qx[:sample1], qy[:sample1], qt[:sample1])
    return r["out64"], dt, sample1 / sec1


def reference_cpu_configs(threads: int, mcl_iterations: int = 10, cfg5_rounds: int = 20) -> dict:
    """The reference's CPU paths beside BASELINE configs 1, 2, 4 and 5 (the
    unmodified rangelib in oracle/_ref, through its public API):
      config 1: Cddt build + 100k casts (one thread, thread cpu time; and all threads)
      config 2: sensor_update (mcl.cpp:58-120), 2,500 particles x 61 paired beams
      config 4: Mcl::step (mcl.cpp:189-201), 40,000 particles x 61 beams, a bounded
                run of `mcl_iterations` steps (its own MclStepResult.seconds)
      config 5: Cddt::set_occupancy over `cfg5_rounds` rounds of 50 random 3x3 blocks
    The reference's sensor model is the analytic beam_likelihood: it has no
    likelihood-table path, so configs 2 and 4 run the analytic model here."""
    import numpy as np

    import oracle
    from paper_1705_01167_b200 import synth
    out = {}
    g1 = synth.rect_map()
    t0 = time.perf_counter()
    r1 = oracle.RefCddt(g1, 108, 300.0)
    build1 = time.perf_counter() - t0
    qx, qy, qt = synth.free_queries(g1, 100_000, seed=7)
    _, sec1 = r1.cast_batch_cpu1(qx, qy, qt)
    t0 = time.perf_counter()
    r1.cast_batch(qx, qy, qt, want_res=False, threads=threads)
    dtn = time.perf_counter() - t0
    out["config1"] = {"build_s": build1, "casts_per_s_1thread": 100_000 / sec1,
                      "casts_per_s_all_threads": 100_000 / dtn, "threads": threads}
    del r1
    g2 = synth.maze_map()
    r2 = oracle.RefCddt(g2, 120, 500.0)
    x, y, t = synth.free_pose(g2, 10, seed=5)
    px, py, pt = synth.particles(x, y, t, 2500, 10.0, 0.1, seed=9)
    scan = synth.scan(g2, x, y, t, 61, 4.71238898038469, 500.0, 8.0, 0.05, seed=13)
    params = oracle.beam_params(sigma_hit=8.0, z_max=500.0)
    r2.sensor_update(px, py, pt, scan, 4.71238898038469, params, paired=True)
    reps, t0 = 5, time.perf_counter()
    for _ in range(reps):
        r2.sensor_update(px, py, pt, scan, 4.71238898038469, params, paired=True)
    ms2 = (time.perf_counter() - t0) / reps * 1e3
    # the table model through the restatement (oracle/cddt_oracle.c, a port), one thread
    from paper_1705_01167_b200 import rangelib
    tab = rangelib.beam_table(rangelib.BeamModelParams(sigma_hit=8.0, z_max=500.0), 501, 1.0)
    o2 = oracle.OracleCddt(g2, 120, 500.0)
    o2.sensor_update(px, py, pt, scan, 4.71238898038469, params, table=tab, threads=1)
    t0 = time.perf_counter()
    for _ in range(reps):
        o2.sensor_update(px, py, pt, scan, 4.71238898038469, params, table=tab, threads=1)
    port = {"ms_per_sensor_update": (time.perf_counter() - t0) / reps * 1e3, "threads": 1}
    del o2
    out["config2"] = {"ms_per_sensor_update": ms2, "casts_per_s": 2500 * 61 / ms2 * 1e3,
                      "threads": 1, "model": "analytic beam_likelihood (no table path in the "
                                               "reference)", "paired_casts": True,
                      "table_model_port": dict(port, kind="port",
                                               what="the 501x501 table model through the C "
                                                    "restatement (oracle/cddt_oracle.c)")}
    x0, y0, t0_ = synth.free_pose(g2, 15, seed=8)
    pose, odo = synth.trajectory(g2, x0, y0, t0_, mcl_iterations, 1.0, 15.0, seed=4)
    scans = np.stack([synth.scan(g2, *pose[k + 1], 61, 4.71238898038469, 500.0, 8.0, 0.05,
                                 seed=1000 + k) for k in range(mcl_iterations)])
    sec, _ = r2.mcl_run(40_000, 5, (x0, y0, t0_), 10.0, 0.1, (1.0, 0.0, 0.0, 0.02), params,
                        4.71238898038469, np.asarray(odo, np.float64), scans)
    out["config4"] = {"ms_per_update_p50": float(np.median(sec)) * 1e3,
                      "ms_per_update_mean": float(np.mean(sec)) * 1e3,
                      "iterations_timed": mcl_iterations, "threads": 1,
                      "extrapolated_1000_iterations_s": float(np.mean(sec)) * 1000,
                      "model": "analytic beam_likelihood (no table path in the reference)",
                      "what": "rangelib::Mcl::step (motion, paired-cast sensor model, estimate, "
                              "resampling), its own MclStepResult.seconds"}
    del r2
    # config 5: the same edit rounds (tests/golden/cfg5_rounds.json's seeds)
    # through the reference's Cddt::set_occupancy, cell by cell in order
    gold = json.loads((ROOT / "tests" / "golden" / "cfg5_rounds.json").read_text())
    r5 = oracle.RefCddt(g2, 108, 0.0)
    sec5 = []
    for r in range(cfg5_rounds):
        xy, occ = synth.block_edits(2000, 2000, 50, seed=gold["seed0"] + r)
        st, sec = r5.set_occupancy_timed(xy, occ)
        if st:
            raise RuntimeError(f"reference set_occupancy failed ({st})")
        sec5.append(sec)
    out["config5"] = {"ms_per_update_round_p50": float(np.median(sec5)) * 1e3,
                      "ms_per_update_round_mean": float(np.mean(sec5)) * 1e3,
                      "rounds_timed": cfg5_rounds, "threads": 1,
                      "what": "rangelib::Cddt::set_occupancy per edited cell (cddt.cpp:332-377), "
                              "the first rounds of the bench's edit sequence, steady clock"}
    return out


def gather_ceiling(device: int) -> dict:
    """Scattered-sector read rates (rl_diag_gather: independent 16-byte reads of
    random 32-byte sectors, full occupancy) out of buffers the size of the
    config-3 query working set (L2) and far beyond L2 (HBM), in G sectors/s."""
    import ctypes as C

    import torch

    from paper_1705_01167_b200._lib import check, lib, torch_stream
    out = {}
    for name, nbytes in (("l2_16MB", 16 << 20), ("l2_111MB", 111 << 20), ("hbm_4GB", 4 << 30)):
        buf = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{device}")
        buf.random_()
        ms, issued = C.c_double(), C.c_uint64()
        check(lib().rl_diag_gather(buf.data_ptr(), nbytes, 1 << 30, torch_stream(buf.device),
                                   C.byref(ms), C.byref(issued)))
        out[name] = issued.value / ms.value / 1e6
        del buf
    return out


def ray_march_cpu(g, qx, qy, qt, sample: int, threads: int) -> dict:
    """The reference's other CPU path for the same queries: make_method(ray_march)
    (proj/src/methods.cpp:55-72), timed on a bounded sample with all threads."""
    import oracle
    oracle.build(ref=True)
    t0 = time.perf_counter()
    rm = oracle.RefRayMarch(g, 1000.0)
    setup = time.perf_counter() - t0
    rm.cast_batch(qx[:10000], qy[:10000], qt[:10000], threads=threads)
    t0 = time.perf_counter()
    rm.cast_batch(qx[:sample], qy[:sample], qt[:sample], threads=threads)
    dt = time.perf_counter() - t0
    return {"value": sample / dt, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{sample} queries of this workload through make_method(ray_march), "
                      f"construction {setup:.2f} s"}


def pf_update_timing(iterations: int, device: int, group=None):
    """BASELINE config 4: full particle-filter update (motion, fused CDDT sensor
    model with the 501x501 table, normalisation, estimate, low-variance
    resampling) for 40,000 particles x 61 beams on the 2000x2000 maze,
    theta_disc 120, max_range 500, along a seeded 1 px/step trajectory.
    With a process group the particles are sharded over its ranks (one GPU
    each; every rank calls this) and the step runs with the two NCCL
    exchanges; per-step times are the max over ranks."""
    import numpy as np
    import torch

    import paper_1705_01167_b200 as rl
    from paper_1705_01167_b200 import mcl, synth
    g = synth.maze_map()
    x, y, t = synth.free_pose(g, 15, seed=8)
    pose, odo = synth.trajectory(g, x, y, t, iterations, 1.0, 15.0, seed=4)
    grid = rl.OccupancyGrid.from_array(g)
    method = rl.make_method("cddt", grid, rl.RangeMethodConfig(500.0, 120), device=device)
    beam = rl.BeamModelParams(sigma_hit=8.0, z_max=500.0)
    table = torch.from_numpy(rl.beam_table(beam, 501, 1.0)).cuda(device)
    cfg = mcl.MclConfig(particle_count=40_000, beam=beam, seed=5,
                        motion=mcl.MotionNoise(1.0, 0.0, 0.0, 0.02))  # sigma_xy 1 px, sigma_th 0.02
    f = mcl.Mcl(method, cfg, table=table, group=group)
    f.init_gaussian(x, y, t, 10.0, 0.1)
    scans = [torch.from_numpy(synth.scan(g, *pose[k + 1], 61, 4.71238898038469, 500.0, 8.0, 0.05,
                                         seed=1000 + k)).cuda(device) for k in range(iterations)]
    for k in range(5):
        f.step(*odo[k], scans[k])
    torch.cuda.synchronize()
    # throughput: the iterations issued back to back (Mcl.step never waits for
    # the device), an event after each; per-update time = consecutive events
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(iterations + 1)]
    evs[0].record()
    results = []
    for k in range(iterations):
        results.append(f.step(*odo[k], scans[k]))
        evs[k + 1].record()
    evs[-1].synchronize()
    times = [evs[k].elapsed_time(evs[k + 1]) for k in range(iterations)]
    errs = [float(np.hypot(r.estimate.x - pose[k + 1][0], r.estimate.y - pose[k + 1][1]))
            for k, r in enumerate(results)]
    # latency: one update at a time, its estimate read back before the next
    lat = []
    for k in range(min(iterations, 100)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = f.step(*odo[k], scans[k])
        r.estimate
        e1.record()
        e1.synchronize()
        lat.append(e0.elapsed_time(e1))
    times = np.array(times)
    world = 1
    if group is not None:
        import torch.distributed as dist
        world = dist.get_world_size(group)
        tt = torch.tensor(times, dtype=torch.float64,
                          device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX, group=group)
        times = tt.cpu().numpy()
    peak, peak_kind = measured_hbm_peak()
    ss = json.loads((ROOT / "profiles" / "sensor_sectors.json").read_text())["config4"]
    b_step = 40_000 * (61 * 32.0 * ss["sectors_per_beam"] + 96.0)
    ach = b_step / (float(np.median(times)) * 1e-3) / 1e9
    roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "peak_source": f"{peak_kind} hbm_gbs",
            "algorithmic_bytes_per_step": b_step,
            "sectors_per_beam": ss["sectors_per_beam"],
            "definition": "SURVEY.md §8d: per particle 61 * 32 * S-bar_beam + 96 B (S-bar_beam from "
                          "the instrumented restatement, profiles/sensor_sectors.json); the sensor "
                          "kernel's working set is cache-resident and it is issue-bound (ncu), so "
                          "this measures how fast the reference's traffic is served"}
    return {"workload": "BASELINE config 4: 40,000 particles x 61 beams, 2000x2000 maze, "
                        f"theta_disc=120, 501x501 table, {world} GPU"
                        + (f"s (particles sharded, {40_000 // world} per GPU; max over ranks)"
                           if world > 1 else ""),
            "iterations": iterations, "ms_per_update_p50": float(np.median(times)),
            "ms_per_update_mean": float(times.mean()), "ms_per_update_p99":
            float(np.percentile(times, 99)),
            "timing": "iterations issued back to back (no host sync), CUDA events between "
                      "updates; ms_per_update_synchronous_p50: one update at a time with its "
                      "estimate read back (host launch latency included)",
            "ms_per_update_synchronous_p50": float(np.median(lat)),
            "roofline": roof,
            "casts_per_update": 40_000 * 61,
            "median_position_error_px": float(np.median(errs[10:]))}


def other_configs(device: int, rounds: int = 1000):
    """BASELINE configs 1, 2 and 5 on one GPU (timings only; parity for each
    is in tests/test_gpu_*.py)."""
    import numpy as np
    import torch

    import paper_1705_01167_b200 as rl
    from paper_1705_01167_b200 import synth
    out = {}

    def ev_time(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    # config 1: 500x500 rectangles, theta_disc 108, max_range 300, 100k queries
    g = synth.rect_map()
    t0 = time.perf_counter()
    c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(300.0, 108), device=device)
    build = time.perf_counter() - t0
    qx, qy, qt = (torch.from_numpy(a).cuda(device) for a in synth.free_queries(g, 100_000, seed=7))
    o = torch.empty_like(qx)
    ms = ev_time(lambda: c.cast_batch(qx, qy, qt, out=o), 200)
    ref = o.clone()
    lat = [ev_time(lambda: c.cast_batch(qx, qy, qt, out=o), 1) for _ in range(50)]
    # the same batches replayed from a CUDA graph (host launch cost removed)
    side = torch.cuda.Stream(device)
    side.wait_stream(torch.cuda.current_stream(device))
    with torch.cuda.stream(side):
        c.cast_batch(qx, qy, qt, out=o)
    torch.cuda.current_stream(device).wait_stream(side)
    graph, per_graph = torch.cuda.CUDAGraph(), 20
    with torch.cuda.graph(graph):
        for _ in range(per_graph):
            c.cast_batch(qx, qy, qt, out=o)
    ms_graph = ev_time(graph.replay, 10) / per_graph
    if not torch.equal(o, ref):
        raise RuntimeError("config 1: graph replay differs from direct calls")
    out["config1"] = {"workload": "500x500 rects, theta_disc=108, max_range=300, CDDT, 100k queries",
                      "build_s": build, "zero_points": c.zero_point_count(),
                      "ms_per_100k_batch": ms, "casts_per_s": 100_000 / ms * 1e3,
                      "ms_per_100k_batch_graphed": ms_graph,
                      "casts_per_s_graphed": 100_000 / ms_graph * 1e3,
                      "single_batch_latency_ms_p50": float(np.median(lat))}
    # config 2: sensor model, 2500 particles x 61 beams, 501x501 table
    g2 = synth.maze_map()
    m2 = rl.make_method("cddt", rl.OccupancyGrid.from_array(g2), rl.RangeMethodConfig(500.0, 120),
                        device=device)
    x, y, t = synth.free_pose(g2, 10, seed=5)
    px, py, pt = synth.particles(x, y, t, 2500, 10.0, 0.1, seed=9)
    scan = torch.from_numpy(synth.scan(g2, x, y, t, 61, 4.71238898038469, 500.0, 8.0, 0.05,
                                       seed=13)).cuda(device)
    beam = rl.BeamModelParams(sigma_hit=8.0, z_max=500.0)
    table = torch.from_numpy(rl.beam_table(beam, 501, 1.0)).cuda(device)
    parts = {k: torch.from_numpy(v).cuda(device) for k, v in
             dict(x=px, y=py, theta=pt, weight=np.zeros_like(px)).items()}
    spec = rl.ScanSpec(61, 4.71238898038469)
    ms2 = ev_time(lambda: rl.sensor_update(parts, m2, scan, spec, beam, table=table), 200)
    flag = torch.zeros(1, dtype=torch.int32, device=f"cuda:{device}")
    ms2a = ev_time(lambda: rl.sensor_update(parts, m2, scan, spec, beam, table=table,
                                            degenerate=flag), 200)
    # the same asynchronous update replayed from a CUDA graph (20 updates per graph)
    side = torch.cuda.Stream(device)
    side.wait_stream(torch.cuda.current_stream(device))
    with torch.cuda.stream(side):
        rl.sensor_update(parts, m2, scan, spec, beam, table=table, degenerate=flag)
    torch.cuda.current_stream(device).wait_stream(side)
    g2graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g2graph):
        for _ in range(20):
            rl.sensor_update(parts, m2, scan, spec, beam, table=table, degenerate=flag)
    ms2g = ev_time(g2graph.replay, 20) / 20
    peak, peak_kind = measured_hbm_peak()
    s2 = json.loads((ROOT / "profiles" / "sensor_sectors.json").read_text())["config2"]
    b_upd = 2500 * (61 * 32.0 * s2["sectors_per_beam"] + 20.0)
    ach2 = b_upd / (ms2a * 1e-3) / 1e9
    out["config2"] = {"workload": "2000x2000 maze, theta_disc=120, max_range=500, 2500 particles x "
                                  "61 beams, 501x501 table",
                      "roofline": {"bound": "hbm", "achieved": ach2, "peak": peak, "unit": "GB/s",
                                   "frac": ach2 / peak, "peak_source": f"{peak_kind} hbm_gbs",
                                   "algorithmic_bytes_per_update": b_upd,
                                   "sectors_per_beam": s2["sectors_per_beam"],
                                   "definition": "SURVEY.md §8d: per beam 32 * S-bar_beam + 20/61 B; "
                                                 "one-wave, latency-bound launch"},
                      "ms_per_sensor_update_graphed": ms2g,
                      "ms_per_sensor_update": ms2a, "casts_per_s": 2500 * 61 / ms2a * 1e3,
                      "timing": "200 updates issued back to back through sensor_update(..., "
                                "degenerate=<device flag>) (rl_sensor_update_async), CUDA events",
                      "ms_per_sensor_update_synchronous": ms2,
                      "synchronous": "sensor_update returning the reference's bool (flag read "
                                     "back every update)"}
    # config 5: 2000x2000 maze, theta_disc 108; 1,000 rounds of 50 random 3x3
    # edits + 1M queries, the round sequence of tests/golden/cfg5_rounds.json
    # (reference digests after every round; tests/test_gpu_cfg5.py checks every
    # one, the bench checks the final structure and casts)
    import hashlib
    gold = json.loads((ROOT / "tests" / "golden" / "cfg5_rounds.json").read_text())
    c5 = rl.Cddt(rl.OccupancyGrid.from_array(g2), rl.RangeMethodConfig(0.0, 108), device=device)
    q5 = [torch.from_numpy(a).cuda(device) for a in synth.free_queries(g2, 1_000_000, seed=31)]
    o5 = torch.empty_like(q5[0])
    edits = [synth.block_edits(2000, 2000, 50, seed=gold["seed0"] + r) for r in range(rounds)]
    upd, qry = [], []
    for r in range(rounds):
        xy, occ = edits[r]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        c5.set_occupancy_batch(xy, occ)
        upd.append(time.perf_counter() - t0)
        qry.append(ev_time(lambda: c5.cast_batch(*q5, out=o5), 1))
    parity = None
    if rounds == len(gold["rounds"]):
        last = gold["rounds"][-1]
        e = c5.export()
        dig = [hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]
               for a in (e["zp"], e["row_off"], e["membership"])]
        o64 = c5.cast_batch_f64(*(a.double() for a in q5))
        parity = (dig == [last["zp"], last["row_off"], last["membership"]]
                  and hashlib.sha256(o64.cpu().numpy().tobytes()).hexdigest() == last["casts"])
    out["config5"] = {"workload": "2000x2000 maze, theta_disc=108, rounds of 50 random 3x3 "
                                  "insert/remove blocks + 1M queries", "rounds": rounds,
                      "ms_per_update_round_p50": 1e3 * float(np.median(upd)),
                      "ms_per_update_round_mean": 1e3 * float(np.mean(upd)),
                      "ms_per_1M_queries_p50": float(np.median(qry)),
                      "zero_points_after": c5.zero_point_count(),
                      "parity_vs_reference_final_round": parity,
                      "parity_note": "zero points, row offsets, membership and 1M f64 casts after "
                                     "the last round equal the reference's digests "
                                     "(tests/golden/cfg5_rounds.json); every round is checked "
                                     "by tests/test_gpu_cfg5.py"}
    return out


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------- arms
def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1705_01167_b200 as rl

    local_rank = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    n = args.queries
    g, qx, qy, qt, np = make_workload(n, rank)
    cddt = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(1000.0, 200),
                   device=local_rank, prune=True)
    info = cddt.info()
    dx, dy, dt = (t.cuda(non_blocking=True) for t in (qx, qy, qt))
    out = torch.empty(n, dtype=torch.float32, device="cuda")
    host_out = torch.empty(n, dtype=torch.float32).pin_memory()
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    with ClockSampler(local_rank) as clk:
        for _ in range(args.warmup):
            cddt.cast_batch(dx, dy, dt, out=out)
        barrier()
        clk.mark()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            cddt.cast_batch(dx, dy, dt, out=out)
        ev1.record(stream)
        barrier()
        t_dev = ev0.elapsed_time(ev1) / 1e3
        # e2e through the host-pointer C-ABI call (pinned H2D + kernel + D2H)
        hx, hy, ht, ho = qx.numpy(), qy.numpy(), qt.numpy(), host_out.numpy()
        for _ in range(max(1, args.warmup // 2)):
            cddt.cast_batch(hx, hy, ht, out=ho)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            cddt.cast_batch(hx, hy, ht, out=ho)
        e1.record(stream)
        barrier()
        t_e2e = e0.elapsed_time(e1) / 1e3
    if world > 1:  # max over ranks
        tt = torch.tensor([t_dev, t_e2e], dtype=torch.float64,
                          device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_dev, t_e2e = tt.tolist()
    if not torch.equal(out.cpu(), host_out):
        raise RuntimeError("device-resident and host-path results differ")

    value = world * n * args.steps / t_dev
    e2e_value = world * n * args.e2e_steps / t_e2e
    e2e_pageable = None
    if rank == 0 and world == 1 and not args.no_extra:
        # the same call with PAGEABLE buffers (what a reference caller holds): staged through
        # a pinned ring by host threads inside the library; the call is synchronous, wall clock
        px, py, pt = (np.array(a, copy=True) for a in (hx, hy, ht))
        po = np.zeros(n, dtype=np.float32)
        cddt.cast_batch(px, py, pt, out=po)
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            cddt.cast_batch(px, py, pt, out=po)
        t_pg = time.perf_counter() - t0
        if not np.array_equal(po, ho):
            raise RuntimeError("pageable and pinned host-path results differ")
        e2e_pageable = {"value": n * args.e2e_steps / t_pg, "unit": UNIT,
                        "path": "rl_cddt_cast_batch_host (pageable numpy buffers, staged through "
                                "a pinned ring by host threads with non-temporal copies)"}
        del px, py, pt, po
    line = None
    sharded_pf = None
    if world > 1 and args.pf_iterations > 0:  # every rank: the sharded filter
        sharded_pf = pf_update_timing(args.pf_iterations, local_rank, group=dist.group.WORLD)
    if rank == 0:
        # GPU extras first: the host-heavy reference sample below leaves CPU
        # worker threads behind that skew host-bound timings
        extras = {}
        if sharded_pf is not None:
            extras["pf_update_sharded"] = sharded_pf
        if args.pf_iterations > 0:
            extras["pf_update"] = pf_update_timing(args.pf_iterations, local_rank)
        if not args.no_extra:
            extras["other_configs"] = other_configs(local_rank)
        peak, peak_kind = measured_hbm_peak()
        sample = min(n, args.cpu_sample)
        threads = os.cpu_count() or 1
        ref, ref_blob, how, same = reference_structure(g)
        # the GPU-built PCDDT, in the reference's snapshot format, byte for byte
        structure_equal = ref_blob is not None and rl.serialize_cddt(cddt) == ref_blob
        ref_out, ref_dt, ref_1t = reference_cpu(ref, qx.numpy(), qy.numpy(), qt.numpy(), sample,
                                                threads, min(n, args.cpu_sample_1t))
        cpu_cfgs = reference_cpu_configs(threads, args.ref_mcl_iterations)
        # parity on the sample: f32 GPU output == float(reference f64)
        got = out[:sample].cpu().numpy()
        mism = int((got != ref_out.astype(np.float32)).sum())
        # algorithmic bytes per query: the reference's sectors per query on this workload,
        # counted by the instrumented restatement in tests/test_gpu_sectors.py
        sectors = json.loads((ROOT / "profiles" / "sectors.json").read_text())
        ns, s_bar = int(sectors["sample"]), float(sectors["sectors_per_query"])
        bytes_per_query = 16.0 + 32.0 * s_bar
        achieved = bytes_per_query * n * args.steps / t_dev / 1e9
        tr = profile_traffic()
        traffic = None
        if tr and tr.get("dram_bytes_per_query"):
            traffic = tr["dram_bytes_per_query"] * n
        # the scattered-read ceiling beside the cast's algorithmic scattered-sector rate
        gather = gather_ceiling(local_rank)
        gather["cast_algorithmic"] = s_bar * n * args.steps / t_dev / 1e9
        gather["frac_of_l2_111MB"] = gather["cast_algorithmic"] / gather["l2_111MB"]
        gather["unit"] = "G sectors/s (random 32-byte sectors; cast: S-bar sectors per query)"
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_dev / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE config-3 map and query stream)",
            "config": dict(workload_config(n), parallelism=f"query-sharded x{world}, structure replicated",
                           dist_backend=(dist.get_backend() if world > 1 else None),
                           zero_points=int(info.zero_points), rows=int(info.rows),
                           device_bytes=int(info.device_bytes),
                           build_plus_prune_s=round(info.init_seconds, 3)),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 12 * n,
                    "d2h_bytes_per_step": 4 * n, "steps": args.e2e_steps,
                    "path": "rl_cddt_cast_batch_host (pinned host buffers, 3-stream pipeline)",
                    "pageable": e2e_pageable},
            # per step: two pipelines (one per half of the batch) of k_cast_defer_p1,
            # k_cast_near and three capped k_walk_pass window passes and the k_walk_last_coop finishing pass
            "gpu_launches": 12 * args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "peak_source": f"{peak_kind} hbm_gbs",
                         "algorithmic_bytes_per_query": bytes_per_query, "sectors_per_query": s_bar,
                         "l2_sectors_per_query": (tr or {}).get("l2_sectors_per_query"),
                         "traffic_source": (tr or {}).get("source"),
                         "sector_sample": ns,
                         "kernel": "batched cast = 2 pipelines (halves of the batch, two streams) of "
                                   "k_cast_defer_p1 + k_cast_near + 3 x k_walk_pass (capped window passes) + k_walk_last_coop (finishing pass); "
                                   "timed per step",
                         "gather_ceiling": gather},
            "cpu_baseline": {"value": sample / ref_dt, "unit": UNIT, "cores": threads,
                             "kind": "reference",
                             "sample": f"{sample} queries of this workload on {how}; "
                                       f"{cpu_model()}",
                             "same_config": same,
                             "gpu_structure_bytes_equal_reference": structure_equal,
                             "value_1thread": ref_1t,
                             "sample_1thread": f"{min(n, args.cpu_sample_1t)} queries on one "
                                               "thread, thread cpu time (the reference's "
                                               "bench.cpp:52-121 clock)",
                             "parity_mismatches": mism,
                             "configs": cpu_cfgs,
                             "ray_march": ray_march_cpu(g, qx.numpy(), qy.numpy(), qt.numpy(),
                                                        min(n, args.rm_sample), threads)},
            "clocks": clk.summary(),
        }
        line.update(extras)
    return line


def run_reference(args):
    """--impl reference: the unmodified reference on the host cores, rank 0 only,
    on the same structure as our arm (the reference-built config-3 PCDDT)."""
    n = args.ref_sample
    g, qx, qy, qt, np = make_workload(n, 0, on_gpu=False)
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    ref, _, how, same = reference_structure(g)
    load_s = time.perf_counter() - t0
    xs, ys, ts = qx.numpy(), qy.numpy(), qt.numpy()
    for _ in range(args.warmup):
        ref.cast_batch(xs, ys, ts, want_res=False, threads=threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ref.cast_batch(xs, ys, ts, want_res=False, threads=threads)
    dt = time.perf_counter() - t0
    value = n * args.steps / dt
    _, sec1 = ref.cast_batch_cpu1(xs[:args.cpu_sample_1t], ys[:args.cpu_sample_1t],
                                  ts[:args.cpu_sample_1t])
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE config-3 map and query stream)",
        "config": dict(workload_config(args.queries), parallelism="host threads"),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": f"{n} queries per step (a bounded sample of the 100M-query "
                                   f"step) on {how} (load {load_s:.1f} s); {cpu_model()}",
                         "same_config": same,
                         "value_1thread": args.cpu_sample_1t / sec1,
                         "sample_1thread": f"{args.cpu_sample_1t} queries on one thread, thread "
                                           "cpu time (the reference's bench.cpp:52-121 clock)",
                         "ray_march": ray_march_cpu(g, xs, ys, ts, min(n, args.rm_sample),
                                                    threads)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` without a launcher: re-run this command under
    torch.distributed.run with N ranks (one per GPU, NCCL, 127.0.0.1), as the
    driver's own torchrun launch would. Refuses when fewer than N GPUs are
    visible rather than timing fewer GPUs than asked for."""
    import socket

    if os.environ.get("BENCH_DIST_BACKEND", "nccl") == "nccl":
        import torch
        have = torch.cuda.device_count()
        if have < n:
            print(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have}", file=sys.stderr)
            return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the init lines show nranks / transports
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "bench.py"),
           *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--queries", type=int, default=100_000_000)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-sample", type=int, default=16_000_000)
    ap.add_argument("--ref-sample", type=int, default=4_000_000)
    ap.add_argument("--cpu-sample-1t", type=int, default=2_000_000,
                    help="queries for the reference's one-thread timing")
    ap.add_argument("--ref-mcl-iterations", type=int, default=20,
                    help="reference Mcl::step iterations timed beside config 4")
    ap.add_argument("--rm-sample", type=int, default=1_000_000,
                    help="queries for the reference's ray-marching CPU timing")
    ap.add_argument("--pf-iterations", type=int, default=1000)
    ap.add_argument("--no-extra", action="store_true", help="skip the config 1/2/5 timings")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return spawn_ranks(args.gpus)
    rank, world, local_rank = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU "
              f"(torchrun --nproc-per-node {args.gpus}) or drop --gpus", file=sys.stderr)
        return 2
    if args.impl == "reference":
        if rank != 0:
            return 0
        print(json.dumps(run_reference(args)), flush=True)
        return 0
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")  # gloo: host-logic checks only
        if backend == "nccl" and local_rank >= torch.cuda.device_count():
            print(f"bench.py: rank {rank} has LOCAL_RANK {local_rank} but only "
                  f"{torch.cuda.device_count()} GPUs are visible", file=sys.stderr)
            return 2
        dev = local_rank % torch.cuda.device_count()  # gloo only: ranks may share a GPU
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    line = run_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
