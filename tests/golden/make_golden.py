"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference
(rangelib compiled from /root/reference/proj/src into oracle/_ref by
oracle/Makefile, driven through oracle/ref_shim.cpp's calls into its public
API). Run in the build container, where the reference sources exist:

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --large    # + full-size hashes (minutes;
                                                  #   the config-3 PCDDT prune is
                                                  #   single-threaded in the reference)

Outputs (committed):
  small.json   exact arrays for small maps: zero points, row offsets,
               membership, cast results (f64 bits) with resolving indices,
               prune results, edit-sequence checkpoints
  large.json   sha256 of the zero-point / row-offset arrays and of cast
               results at the BASELINE config sizes
"""
from __future__ import annotations

import hashlib
import json
import sys
import time
import zlib
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_1705_01167_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def splitmix_random_map(w, h, density, seed):
    """make_random_map (proj/src/synthetic.cpp:84-93), restated bit-exactly."""
    m = (1 << 64) - 1
    st = seed & m
    out = np.zeros(w * h, np.uint8)
    for i in range(w * h):
        st = (st + 0x9E3779B97F4A7C15) & m
        z = st
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
        z ^= z >> 31
        out[i] = 1 if (z >> 11) * 2.0 ** -53 < density else 0
    return out.reshape(h, w)


def structure(ref, full_limit: int = 20000) -> dict:
    """Exact arrays for small structures, sha256 digests for larger ones."""
    e = ref.export()
    i = ref.info()
    d = dict(info=i, zp_sha=sha(e["zp"]), row_off_sha=sha(e["row_off"]),
             membership_sha=sha(e["membership"]))
    if i["zero_points"] <= full_limit:
        d.update(row_off=e["row_off"].tolist(), zp_bits=e["zp"].view(np.uint32).tolist(),
                 membership=np.packbits(e["membership"].ravel()).tolist())
    return d


def small() -> dict:
    maps = {}
    fig4 = np.zeros((4, 4), np.uint8)
    fig4[0, 3] = fig4[1, 1] = fig4[2, 2] = fig4[3, 3] = 1
    cases = [
        ("fig4_k8", fig4, 8, 0.0),
        ("rand64_s1000_k216", splitmix_random_map(64, 64, 0.08, 1000), 216, 0.0),
        ("rand64_s1001_k108", splitmix_random_map(64, 64, 0.08, 1001), 108, 0.0),
        ("rand37x5_k24", splitmix_random_map(37, 5, 0.2, 7), 24, 0.0),
        ("rect96_k36_mr40", synth.rect_map(96, 96, 6, seed=4), 36, 40.0),
    ]
    rng = np.random.default_rng(20260101)
    for name, g, K, mr in cases:
        h, w = g.shape
        ref = oracle.RefCddt(g, K, mr)
        n = 600
        qx = rng.uniform(-1.0, w + 1.0, n).astype(np.float32)
        qy = rng.uniform(-1.0, h + 1.0, n).astype(np.float32)
        qt = rng.uniform(-7.0, 14.0, n).astype(np.float32)
        r = ref.cast_batch(qx, qy, qt)
        entry = dict(grid=np.packbits(g.ravel()).tolist(), w=w, h=h, theta_disc=K, max_range=mr,
                     max_range_resolved=ref.max_range(), cddt=structure(ref),
                     queries=dict(x=qx.view(np.uint32).tolist(), y=qy.view(np.uint32).tolist(),
                                  t=qt.view(np.uint32).tolist()),
                     casts=dict(out64=r["out64"].view(np.uint64).astype(str).tolist(),
                                res_row=r["res_row"].tolist(), res_idx=r["res_idx"].tolist()))
        if w * h <= 4096:
            p = oracle.RefCddt(g, K, mr, prune=True)
            entry["pcddt"] = structure(p)
        # an edit sequence, checkpointed
        if name.startswith("rand64") or name == "rand37x5_k24":
            e_rng = np.random.default_rng(zlib.crc32(name.encode()))
            edits, checkpoints = [], []
            for k in range(40):
                x, y, o = int(e_rng.integers(0, w)), int(e_rng.integers(0, h)), int(e_rng.integers(0, 2))
                ref.set_occupancy(x, y, bool(o))
                edits.append([x, y, o])
                if k % 10 == 9:
                    e = ref.export()
                    checkpoints.append(dict(after=k + 1, zero_points=ref.info()["zero_points"],
                                            zp_sha=sha(e["zp"]), row_off_sha=sha(e["row_off"]),
                                            membership_sha=sha(e["membership"])))
            entry["edits"] = dict(seq=edits, checkpoints=checkpoints)
        maps[name] = entry
    # reference unit-test fixtures (proj/tests/test_cddt.cpp:349-360, :445-462)
    fixtures = dict(
        fig4_casts=[[0.5, 0.5, 0.0, 3.0], [2.5, 1.5, 0.0, "mr"], [2.5, 0.5, "pi", "mr"],
                    [3.7, 1.5, "pi", 2.2], [3.7, 2.5, "pi", 0.7], [1.5, 1.5, 0.3, 0.0],
                    [-0.5, 1.5, 0.0, "mr"], [0.5, 4.5, 0.0, "mr"]],
        fig4_bins_slice0=[[3.5], [1.5], [2.5], [3.5], []],
        corridor_pair=[[2.5, 0.5, 0.0, 2.0, 2.0]],
    )
    return dict(generator="tests/golden/make_golden.py (reference via oracle/_ref)", maps=maps,
                fixtures=fixtures)


def large() -> dict:
    out = {}

    def record(name, g, K, mr, prune, nq, qseed):
        t0 = time.time()
        ref = oracle.RefCddt(g, K, mr, prune=prune)
        e = ref.export()
        rec = dict(theta_disc=K, max_range=mr, pruned=prune, info=ref.info(),
                   zp_sha=sha(e["zp"]), row_off_sha=sha(e["row_off"]),
                   membership_sha=sha(e["membership"]), build_s=round(time.time() - t0, 2))
        if nq:
            qx, qy, qt = synth.free_queries(g, nq, seed=qseed)
            r = ref.cast_batch(qx, qy, qt, want_res=False, threads=8)["out64"]
            rec.update(queries=nq, query_seed=qseed, casts_sha=sha(r),
                       casts_f32_sha=sha(r.astype(np.float32)))
        out[name] = rec
        print(name, rec["info"], rec["build_s"], flush=True)
        return ref

    g1 = synth.rect_map()
    record("cfg1_cddt", g1, 108, 300.0, False, 100_000, 7)
    record("cfg1_pcddt", g1, 108, 300.0, True, 100_000, 7)
    g2 = synth.maze_map()
    record("cfg2_cddt", g2, 120, 500.0, False, 1_000_000, 21)
    # config 5: maze map, theta_disc 108, three edit rounds
    ref5 = record("cfg5_cddt", g2, 108, 0.0, False, 0, 0)
    rounds = []
    for rnd in range(3):
        xy, occ = synth.block_edits(2000, 2000, 50, seed=500 + rnd)
        for (x, y), o in zip(xy, occ):
            ref5.set_occupancy(int(x), int(y), bool(o))
        e = ref5.export()
        rounds.append(dict(seed=500 + rnd, zero_points=ref5.info()["zero_points"],
                           zp_sha=sha(e["zp"]), row_off_sha=sha(e["row_off"]),
                           membership_sha=sha(e["membership"])))
    out["cfg5_rounds"] = rounds
    g3 = synth.polygon_map()
    record("cfg3_cddt", g3, 200, 1000.0, False, 1_000_000, 7)
    record("cfg3_pcddt", g3, 200, 1000.0, True, 1_000_000, 7)
    return out


if __name__ == "__main__":
    oracle.build(ref=True)
    s = small()
    (OUT / "small.json").write_text(json.dumps(s, separators=(",", ":")))
    print("small.json", (OUT / "small.json").stat().st_size)
    if "--large" in sys.argv:
        lg = large()
        (OUT / "large.json").write_text(json.dumps(lg, indent=1))
        print("large.json written")
