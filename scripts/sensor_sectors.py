"""Algorithmic bytes of the sensor model: the mean number of
distinct 32-byte sectors the reference algorithm touches per beam cast (S̄_beam),
counted by the instrumented restatement (oracle/cddt_oracle.c) on the config-2
update (2,500 particles x 61 beams) and on the config-4 initial cloud (40,000
particles x 61 beams), rays rounded to f32 for the restatement's batch entry.
Writes profiles/sensor_sectors.json, which bench.py reads for the config-2 and
config-4 rooflines:
  B_update(config 2) = n * (61 * 32 * S̄_beam + 20) bytes,
  B_step(config 4)   = n * (61 * 32 * S̄_beam + 96) bytes.

    python scripts/sensor_sectors.py
"""
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_1705_01167_b200 import synth  # noqa: E402

FOV = 4.71238898038469


def beams(px, py, pt, nb=61):
    off = np.array([-FOV / 2.0 + FOV * b / (nb - 1) for b in range(nb)])
    th = (pt[:, None] + off[None, :]).ravel()
    return (np.repeat(px, nb).astype(np.float32), np.repeat(py, nb).astype(np.float32),
            np.mod(th, 2 * math.pi).astype(np.float32))


if __name__ == "__main__":
    g = synth.maze_map()
    orc = oracle.OracleCddt(g, 120, 500.0)
    out = {"definition": "mean distinct 32-byte sectors the reference algorithm touches per beam "
                         "cast under the reference layout (oracle/cddt_oracle.c)",
           "generator": "scripts/sensor_sectors.py"}
    x, y, t = synth.free_pose(g, 10, seed=5)
    px, py, pt = synth.particles(x, y, t, 2500, 10.0, 0.1, seed=9)
    sec = orc.cast_batch(*beams(px, py, pt), want_f64=False, want_hit=False, want_res=False,
                         want_sectors=True)["sectors"]
    out["config2"] = {"particles": 2500, "beams": 61, "sectors_per_beam": float(np.mean(sec))}
    x, y, t = synth.free_pose(g, 15, seed=8)
    rng = np.random.Generator(np.random.Philox(key=5))
    n = 40_000
    px = x + 10.0 * rng.standard_normal(n)
    py = y + 10.0 * rng.standard_normal(n)
    pt = np.mod(t + 0.1 * rng.standard_normal(n), 2 * math.pi)
    sec = orc.cast_batch(*beams(px, py, pt), want_f64=False, want_hit=False, want_res=False,
                         want_sectors=True)["sectors"]
    out["config4"] = {"particles": n, "beams": 61, "sectors_per_beam": float(np.mean(sec)),
                      "cloud": "Mcl.init_gaussian(pose, 10 px, 0.1 rad), seed 5 (the bench's start)"}
    (ROOT / "profiles" / "sensor_sectors.json").write_text(json.dumps(out, indent=1))
    print(json.dumps(out, indent=1))
