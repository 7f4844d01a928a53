"""Per-round golden digests for BASELINE config 5 (online map updates), from
the UNMODIFIED reference (oracle/_ref): the 2000x2000 maze map, theta_disc 108,
1,000 rounds, round r applying synth.block_edits(2000, 2000, 50,
seed=500 + r) (50 random 3x3 insert/remove blocks, 450 pixel edits) through
the reference's Cddt::set_occupancy (proj/src/cddt.cpp:332-377), one call per
pixel, in order.

After EVERY round it records the zero-point count and a digest of the
zero-point array, the CSR row offsets and the membership bitmap (the first 32
hex digits of sha256 over the exported arrays, as tests/golden/large.json's
full digests); every 100 rounds also the sha256 of the reference's f64 casts of
1M free-space queries (synth.free_queries(map, 1M, seed=31), the bench's
config-5 stream). Rounds 0-2 equal large.json's cfg5_rounds.

    python tests/golden/make_cfg5_golden.py      # ~15-20 min on 8 cores

Output (committed): tests/golden/cfg5_rounds.json
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_1705_01167_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent / "cfg5_rounds.json"
ROUNDS, SEED0, CAST_EVERY, NQ, QSEED = 1000, 500, 100, 1_000_000, 31


def dig(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def main(rounds: int = ROUNDS) -> None:
    oracle.build(ref=True)
    g = synth.maze_map()
    ref = oracle.RefCddt(g, 108, 0.0)
    qx, qy, qt = synth.free_queries(g, NQ, seed=QSEED)
    out = dict(generator="tests/golden/make_cfg5_golden.py (reference via oracle/_ref)",
               map="synth.maze_map()", theta_disc=108, max_range=0.0, seed0=SEED0,
               edits="synth.block_edits(2000, 2000, 50, seed=seed0 + round)",
               digest="sha256(array bytes)[:32]; zp f32, row_off u64, membership u8 [h, w]",
               queries=dict(n=NQ, seed=QSEED, every=CAST_EVERY,
                            digest="sha256 of the reference's f64 casts (after the round)"),
               rounds=[])
    t0 = time.time()
    for r in range(rounds):
        xy, occ = synth.block_edits(2000, 2000, 50, seed=SEED0 + r)
        for (x, y), o in zip(xy, occ):
            ref.set_occupancy(int(x), int(y), bool(o))
        e = ref.export()
        rec = dict(r=r, edits=int(len(occ)), zero_points=int(e["zp"].size), zp=dig(e["zp"]),
                   row_off=dig(e["row_off"]), membership=dig(e["membership"]))
        if (r + 1) % CAST_EVERY == 0:
            c = ref.cast_batch(qx, qy, qt, want_res=False, threads=8)["out64"]
            rec["casts"] = hashlib.sha256(c.tobytes()).hexdigest()
        out["rounds"].append(rec)
        if r % 50 == 0:
            print(f"round {r} zp={rec['zero_points']} {time.time() - t0:.0f}s", flush=True)
    OUT.write_text(json.dumps(out, separators=(",", ":")))
    print(OUT, OUT.stat().st_size, f"{time.time() - t0:.0f}s")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else ROUNDS)
