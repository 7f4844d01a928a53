"""Helper for tests/test_gpu_sensor.py::test_paired_beams_bitwise: log-weights
of the fused sensor kernel (rl_sensor_logw) on a battery of particle sets and
scan layouts, saved to an .npz. Run once with RL_SENSOR_PAIRED=1 (paired
beams share a row search) and once with RL_SENSOR_PAIRED=0 (every beam its
own cast); the outputs must be byte-identical.

    RL_SENSOR_PAIRED=0 python tests/sensor_pair_probe.py out.npz
"""
import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1705_01167_b200 as rl  # noqa: E402
from paper_1705_01167_b200 import synth  # noqa: E402


def particles(g, n, seed, K):
    h, w = g.shape
    rng = np.random.default_rng(seed)
    x0, y0, t0 = synth.free_pose(g, 10, seed=seed)
    px, py, pt = synth.particles(x0, y0, t0, n, 30.0, 3.0, seed=seed)
    k = n // 8
    # uniform over the whole map (occupied origins, non-clear origins near walls)
    px[:k] = rng.uniform(0, w, k)
    py[:k] = rng.uniform(0, h, k)
    pt[:k] = rng.uniform(-7, 14, k)
    # off the map
    px[k:k + 16] = rng.uniform(-50, -0.001, 16)
    py[k + 16:k + 32] = h + rng.uniform(0, 50, 16)
    # headings on the direction lattice and half-way between (pairing edge cases)
    j = np.arange(2 * k, 3 * k)
    pt[j] = (j % K) * (2 * math.pi / K) + np.where(j % 2 == 0, 0.0, math.pi / K)
    # integer / half-integer origins (projections exactly representable)
    px[3 * k:4 * k] = np.round(px[3 * k:4 * k])
    py[3 * k:4 * k] = np.round(py[3 * k:4 * k]) + 0.5
    return px, py, pt


def main(out):
    res = {}
    for name, g, K, mr in (("maze120", synth.maze_map(), 120, 500.0),
                           ("rect108", synth.rect_map(), 108, 300.0),
                           ("maze16", synth.maze_map(400, 400, 0.1, 4), 16, 0.0)):
        method = rl.make_method("cddt", rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(mr, K))
        mrr = method.max_range()
        beam = rl.BeamModelParams(sigma_hit=8.0, z_max=mrr)
        table = torch.from_numpy(rl.beam_table(beam, 301, 1.0)).cuda()
        for n in (3000, 20000):
            px, py, pt = particles(g, n, 100 + n, K)
            parts = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in
                     dict(x=px, y=py, theta=pt, weight=np.zeros(n)).items()}
            for nb, fov in ((61, 4.71238898038469), (2, math.pi), (90, 2 * math.pi), (1, 0.0),
                            (7, 3.0), (121, 6.0), (40, math.pi + 0.05)):
                rng = np.random.default_rng(nb)
                scan = torch.from_numpy(rng.uniform(0, mrr, nb)).cuda()
                lw = torch.empty(n, dtype=torch.float64, device="cuda")
                rl.sensor_update(parts, method, scan, rl.ScanSpec(nb, fov), beam,
                                 table=table if nb % 2 else None, logw=lw)
                res[f"{name}_{n}_{nb}"] = lw.cpu().numpy()
    np.savez(out, **res)


if __name__ == "__main__":
    main(sys.argv[1])
