"""GPU: BASELINE config 5 at full length — the 2000x2000 maze, theta_disc 108,
1,000 rounds of 50 random 3x3 insert/remove blocks applied through the
incremental update (rl_cddt_set_occupancy_batch), with the zero-point array,
the CSR row offsets and the membership bitmap bit-exact against the reference
after EVERY round, and the f64 casts of 1M free-space queries bit-exact every
100 rounds (digests from the unmodified reference's sequential
Cddt::set_occupancy, proj/src/cddt.cpp:332-377, recorded by
tests/golden/make_cfg5_golden.py)."""
import hashlib
import json
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden" / "cfg5_rounds.json"


def _dig(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


@pytest.mark.timeout(1800)
def test_cfg5_1000_rounds_every_round_vs_reference(rl, synth):
    import torch
    gold = json.loads(GOLD.read_text())
    rounds = gold["rounds"]
    assert len(rounds) == 1000
    g = synth.maze_map()
    c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(gold["max_range"],
                                                                      gold["theta_disc"]))
    q = gold["queries"]
    qx, qy, qt = (torch.from_numpy(a.astype(np.float64)).cuda()
                  for a in synth.free_queries(g, q["n"], seed=q["seed"]))
    pool = ThreadPoolExecutor(3)
    bad = []
    for rd in rounds:
        xy, occ = synth.block_edits(2000, 2000, 50, seed=gold["seed0"] + rd["r"])
        assert len(occ) == rd["edits"]
        c.set_occupancy_batch(xy, occ)
        assert c.zero_point_count() == rd["zero_points"], rd["r"]
        e = c.export()
        digs = pool.map(_dig, (e["zp"], e["row_off"], e["membership"]))
        if tuple(digs) != (rd["zp"], rd["row_off"], rd["membership"]):
            bad.append(rd["r"])
        if "casts" in rd:
            out = c.cast_batch_f64(qx, qy, qt)
            got = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()
            assert got == rd["casts"], f"casts differ after round {rd['r']}"
    assert not bad, f"structure differs from the reference after rounds {bad[:10]}"
