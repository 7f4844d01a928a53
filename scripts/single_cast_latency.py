"""Per-ray latency of the reference-facing single-query entry points
(rl_cddt_cast / rl_cddt_cast_pair: one tiny kernel + one stream sync per call,
the path rangelib::RangeMethod::cast callers such as sensor_update take through
include/rl_cddt_rangemethod.hpp), beside the reference's own per-ray cost on
the host (Cddt::cast, one thread). Config 1 map (500x500, theta_disc 108).

    python scripts/single_cast_latency.py
"""
import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_1705_01167_b200 as rl  # noqa: E402
from paper_1705_01167_b200 import _lib, synth  # noqa: E402

g = synth.rect_map()
c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(300.0, 108))
qx, qy, qt = synth.free_queries(g, 20000, seed=7)
L = _lib.lib()
out, o2 = C.c_double(), C.c_double()
for i in range(200):
    L.rl_cddt_cast(c.handle, float(qx[i]), float(qy[i]), float(qt[i]), C.byref(out))
res = {}
for name, fn in (("cast", lambda i: L.rl_cddt_cast(c.handle, float(qx[i]), float(qy[i]),
                                                   float(qt[i]), C.byref(out))),
                 ("cast_pair", lambda i: L.rl_cddt_cast_pair(c.handle, float(qx[i]), float(qy[i]),
                                                             float(qt[i]), C.byref(out),
                                                             C.byref(o2)))):
    t0 = time.perf_counter()
    for i in range(20000):
        fn(i)
    res[f"us_per_{name}"] = (time.perf_counter() - t0) / 20000 * 1e6
try:
    import oracle
    ref = oracle.RefCddt(g, 108, 300.0)
    _, sec = ref.cast_batch_cpu1(qx, qy, qt)
    res["reference_us_per_cast_1thread"] = sec / 20000 * 1e6
except Exception as e:  # noqa: BLE001
    res["reference"] = f"unavailable: {e}"
print(json.dumps(res))
