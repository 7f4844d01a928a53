"""GPU parity: construction, queries, pruning, edits and snapshots of the CUDA
CDDT against the unmodified reference (oracle/_ref) and the C restatement
(oracle/), on the same seeded inputs. Bit-exact everywhere: zero-point arrays,
row offsets, membership, FP64 ranges, hit cells and resolving indices."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


def fig4():
    # proj/tests/support/oracles.hpp:19-26
    g = np.zeros((4, 4), np.uint8)
    g[0, 3] = g[1, 1] = g[2, 2] = g[3, 3] = 1
    return g


def random_map(w, h, density, seed):
    # make_random_map (proj/src/synthetic.cpp:84-93): SplitMix64 uniform < density
    s = np.uint64(seed)
    out = np.zeros(w * h, np.uint8)
    m64 = (1 << 64) - 1
    st = seed & m64
    for i in range(w * h):
        st = (st + 0x9E3779B97F4A7C15) & m64
        z = st
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m64
        z ^= z >> 31
        out[i] = 1 if (z >> 11) * 2.0 ** -53 < density else 0
    del s
    return out.reshape(h, w)


def make_gpu(rl, g, K, max_range=0.0, prune=False):
    grid = rl.OccupancyGrid.from_array(g)
    return rl.Cddt(grid, rl.RangeMethodConfig(max_range, K), prune=prune)


def assert_same_structure(gpu, ref_export):
    e = gpu.export()
    assert np.array_equal(e["row_off"], ref_export["row_off"])
    assert np.array_equal(e["zp"].view(np.uint32), ref_export["zp"].view(np.uint32))
    assert np.array_equal(e["membership"], ref_export["membership"])


def test_fig4_bins_and_fixtures(rl):
    # proj/tests/test_cddt.cpp:229-242 and :349-360
    c = make_gpu(rl, fig4(), 8)
    assert c.theta_disc() == 8 and c.slice_count() == 4
    assert c.max_range() == pytest.approx(math.sqrt(32.0))
    assert c.slice(0).bin_count == 5
    assert c.bin(0, 0).values() == [3.5]
    assert c.bin(0, 1).values() == [1.5]
    assert c.bin(0, 2).values() == [2.5]
    assert c.bin(0, 3).values() == [3.5]
    assert c.bin(0, 4).empty()
    mr = c.max_range()
    Q = rl.RayQuery
    assert c.cast(Q(0.5, 0.5, 0.0)) == pytest.approx(3.0)
    assert c.cast(Q(2.5, 1.5, 0.0)) == pytest.approx(mr)
    assert c.cast(Q(2.5, 0.5, rl.kTwoPi / 2.0)) == pytest.approx(mr)
    assert c.cast(Q(3.7, 1.5, rl.kTwoPi / 2.0)) == pytest.approx(2.2)
    assert c.cast(Q(3.7, 2.5, rl.kTwoPi / 2.0)) == pytest.approx(0.7)
    assert c.cast(Q(1.5, 1.5, 0.3)) == pytest.approx(0.0)
    assert c.cast(Q(-0.5, 1.5, 0.0)) == pytest.approx(mr)
    assert c.cast(Q(0.5, 4.5, 0.0)) == pytest.approx(mr)


def test_corridor_cast_pair(rl):
    # proj/tests/test_cddt.cpp:445-462
    g = np.zeros((1, 5), np.uint8)
    g[0, 0] = g[0, 4] = 1
    c = make_gpu(rl, g, 8)
    f, b = c.cast_pair(rl.RayQuery(2.5, 0.5, 0.0))
    assert f == pytest.approx(2.0) and b == pytest.approx(2.0)
    g2 = np.zeros((1, 5), np.uint8)
    g2[0, 4] = 1
    c2 = make_gpu(rl, g2, 8)
    f, b = c2.cast_pair(rl.RayQuery(1.5, 0.5, 0.0))
    assert f == pytest.approx(3.0) and b == pytest.approx(c2.max_range())


def test_config_validation_errors(rl):
    grid = rl.OccupancyGrid.from_array(fig4())
    with pytest.raises(ValueError):
        rl.Cddt(grid, rl.RangeMethodConfig(0.0, 7))
    with pytest.raises(ValueError):
        rl.Cddt(grid, rl.RangeMethodConfig(-1.0, 8))


def test_empty_grid(rl):
    # proj/tests/test_cddt.cpp:244-250
    c = make_gpu(rl, np.zeros((9, 12), np.uint8), 12)
    assert c.zero_point_count() == 0
    assert c.cast(rl.RayQuery(6.0, 4.5, 1.0)) == pytest.approx(c.max_range())


@pytest.mark.parametrize("case", ["fig4", "rand64", "rand_ragged", "full", "cfg1", "line"])
def test_build_bitexact_vs_reference(rl, oracle_mod, synth, case):
    K, mr = 108, 0.0
    if case == "fig4":
        g, K = fig4(), 8
    elif case == "rand64":
        g, K = random_map(64, 64, 0.08, 1001), 216
    elif case == "rand_ragged":
        g, K = random_map(37, 5, 0.2, 7), 24
    elif case == "full":
        g, K = np.ones((16, 9), np.uint8), 12
    elif case == "line":
        g, K = np.zeros((20, 20), np.uint8), 16
        g[7, 5:15] = 1
    else:
        g, K, mr = synth.rect_map(), 108, 300.0
    gpu = make_gpu(rl, g, K, mr)
    ref = (oracle_mod.RefCddt if oracle_mod.ref_available() else oracle_mod.OracleCddt)(g, K, mr)
    assert gpu.info().rows == ref.info()["rows"]
    assert gpu.zero_point_count() == ref.info()["zero_points"]
    assert gpu.memory_bytes() == ref.info()["memory_bytes"]
    assert_same_structure(gpu, ref.export())


def test_casts_bitexact_cfg1(rl, oracle_mod, synth):
    import torch
    g = synth.rect_map()
    gpu = make_gpu(rl, g, 108, 300.0)
    qx, qy, qt = synth.free_queries(g, 100_000, seed=7)
    orc = oracle_mod.OracleCddt(g, 108, 300.0).cast_batch(qx, qy, qt)
    # f64 path with hit cell and resolving index
    x, y, t = (dev(a.astype(np.float64)) for a in (qx, qy, qt))
    n = qx.size
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    hit = torch.empty(n, dtype=torch.int32, device="cuda")
    rr = torch.empty(n, dtype=torch.int64, device="cuda")
    ri = torch.empty(n, dtype=torch.int32, device="cuda")
    gpu.cast_batch_f64(x, y, t, out, hit, rr, ri)
    torch.cuda.synchronize()
    assert np.array_equal(host(out).view(np.uint64), orc["out64"].view(np.uint64))
    assert np.array_equal(host(hit), orc["hit"])
    assert np.array_equal(host(rr), orc["res_row"])
    assert np.array_equal(host(ri), orc["res_idx"])
    if oracle_mod.ref_available():
        ref = oracle_mod.RefCddt(g, 108, 300.0).cast_batch(qx, qy, qt)
        assert np.array_equal(host(out).view(np.uint64), ref["out64"].view(np.uint64))
        assert np.array_equal(host(rr), ref["res_row"])
        assert np.array_equal(host(ri), ref["res_idx"])
    # f32 device path == float(reference f64)
    o32 = gpu.cast_batch(dev(qx), dev(qy), dev(qt), hit=hit)
    torch.cuda.synchronize()
    assert np.array_equal(host(o32), orc["out64"].astype(np.float32))
    assert np.array_equal(host(hit), orc["hit"])
    # host pipelined path
    oh = gpu.cast_batch(qx, qy, qt)
    assert np.array_equal(oh, orc["out32"])


def test_casts_edge_inputs(rl, oracle_mod):
    """Off-map, on-lattice, exact-axis, huge/negative angles, zero-length batch."""
    import torch
    g = random_map(48, 40, 0.1, 99)
    gpu = make_gpu(rl, g, 24, 0.0)
    orc = oracle_mod.OracleCddt(g, 24, 0.0)
    rng = np.random.default_rng(3)
    xs = np.concatenate([rng.uniform(-2, 50, 2000), np.arange(0, 48, 0.5), [-0.0, 48.0, 47.999]])
    ys = np.concatenate([rng.uniform(-2, 42, 2000), np.arange(0, 40, 40 / 96), [0.0, 39.99, 40.0]])
    n = min(xs.size, ys.size)
    xs, ys = xs[:n].astype(np.float32), ys[:n].astype(np.float32)
    ts = np.concatenate([rng.uniform(-20, 20, n - 8),
                         [0, np.pi / 2, np.pi, 3 * np.pi / 2, 2 * np.pi, -1e-7, 1e4, -1e4]])
    ts = ts.astype(np.float32)
    want = orc.cast_batch(xs, ys, ts)
    got = gpu.cast_batch(dev(xs), dev(ys), dev(ts))
    torch.cuda.synchronize()
    assert np.array_equal(host(got), want["out32"])
    empty = torch.empty(0, dtype=torch.float32, device="cuda")
    gpu.cast_batch(empty, empty, empty)


def test_cast_pair_equals_two_casts(rl, oracle_mod):
    # proj/tests/test_cddt.cpp:430-443
    g = random_map(32, 32, 0.1, 3)
    gpu = make_gpu(rl, g, 24)
    rng = np.random.default_rng(7)
    for _ in range(50):
        q = rl.RayQuery(rng.uniform(-1, 33), rng.uniform(-1, 33), rng.uniform(0, rl.kTwoPi))
        f, b = gpu.cast_pair(q)
        assert f == gpu.cast(q)
        assert b == gpu.cast(rl.RayQuery(q.x, q.y, q.theta + rl.kTwoPi / 2.0))


@pytest.mark.parametrize("case", ["rand20", "line", "block", "cfg1"])
def test_prune_bitexact(rl, oracle_mod, synth, case):
    K, mr = 16, 0.0
    if case == "rand20":
        g = random_map(20, 20, 0.1, 51)
    elif case == "line":
        g = np.zeros((20, 20), np.uint8)
        g[7, 5:15] = 1
    elif case == "block":
        g, K = np.zeros((5, 5), np.uint8), 8
        g[1:4, 1:4] = 1
    else:
        g, K, mr = synth.rect_map(), 108, 300.0
    gpu = make_gpu(rl, g, K, mr, prune=True)
    assert gpu.pruned()
    ref = (oracle_mod.RefCddt if oracle_mod.ref_available() else oracle_mod.OracleCddt)(
        g, K, mr, prune=True)
    assert gpu.zero_point_count() == ref.info()["zero_points"]
    assert_same_structure(gpu, ref.export())
    if case == "line":
        assert gpu.bin(0, 7).size() <= 2  # proj/tests/test_cddt.cpp:503-512
    with pytest.raises(rl.LogicError):
        gpu.set_occupancy(0, 0, True)


def test_prune_preserves_discrete_states(rl, oracle_mod):
    # proj/tests/test_cddt.cpp:464-484 on the GPU: PCDDT == CDDT at every
    # (cell centre, direction) state
    import torch
    g = random_map(24, 24, 0.1, 53)
    K = 16
    full = make_gpu(rl, g, K)
    pr = make_gpu(rl, g, K, prune=True)
    ys, xs, aa = np.meshgrid(np.arange(24), np.arange(24), np.arange(K), indexing="ij")
    x = dev(xs.ravel().astype(np.float64) + 0.5)
    y = dev(ys.ravel().astype(np.float64) + 0.5)
    a = dev(aa.ravel().astype(np.int32))
    r0 = full.directional_batch(x, y, a)
    r1 = pr.directional_batch(x, y, a)
    torch.cuda.synchronize()
    assert torch.equal(r0, r1)


def test_set_occupancy_errors(rl):
    c = make_gpu(rl, fig4(), 8)
    with pytest.raises(IndexError):
        c.set_occupancy(-1, 0, True)
    with pytest.raises(IndexError):
        c.set_occupancy(0, 4, True)
    n = c.zero_point_count()
    c.set_occupancy(1, 1, True)  # already occupied: no-op
    c.set_occupancy(0, 0, False)
    assert c.zero_point_count() == n


def test_edits_match_reference_sequence(rl, oracle_mod):
    # proj/tests/test_cddt.cpp:578-604: random edits, compared after each batch
    g = random_map(16, 16, 0.1, 14)
    K = 8
    gpu = make_gpu(rl, g, K)
    ref = (oracle_mod.RefCddt if oracle_mod.ref_available() else oracle_mod.OracleCddt)(g, K)
    rng = np.random.default_rng(1000)
    for rnd in range(6):
        xy = rng.integers(0, 16, size=(10, 2)).astype(np.int32)
        occ = rng.integers(0, 2, size=10).astype(np.uint8)
        for (x, y), o in zip(xy, occ):
            ref.set_occupancy(int(x), int(y), bool(o))
        if rnd % 2:
            gpu.set_occupancy_batch(xy, occ)
        else:
            for (x, y), o in zip(xy, occ):
                gpu.set_occupancy(int(x), int(y), bool(o))
        assert gpu.zero_point_count() == ref.info()["zero_points"]
        assert_same_structure(gpu, ref.export())


def test_block_edit_rounds_maze(rl, oracle_mod, synth):
    """Config-5 style rounds (3x3 insert/remove blocks) on a 400x400 maze:
    structure bit-exact with the sequential oracle after every round, and
    equal to a fresh GPU build of the edited grid."""
    g = synth.maze_map(400, 400, 0.10, 5)
    K = 108
    gpu = make_gpu(rl, g, K)
    orc = oracle_mod.OracleCddt(g, K)
    for rnd in range(5):
        xy, occ = synth.block_edits(400, 400, 50, seed=100 + rnd)
        for (x, y), o in zip(xy, occ):
            orc.set_occupancy(int(x), int(y), bool(o))
        gpu.set_occupancy_batch(xy, occ)
        assert_same_structure(gpu, orc.export())
    fresh = make_gpu(rl, gpu.export()["grid"], K)
    assert_same_structure(gpu, fresh.export())


def test_edit_batch_prefix_on_error(rl, oracle_mod):
    g = random_map(16, 16, 0.1, 4)
    gpu = make_gpu(rl, g, 8)
    orc = oracle_mod.OracleCddt(g, 8)
    xy = np.array([[3, 3], [5, 5], [99, 1], [6, 6]], np.int32)
    occ = np.array([1, 1, 1, 1], np.uint8)
    with pytest.raises(IndexError):
        gpu.set_occupancy_batch(xy, occ)
    orc.set_occupancy(3, 3, True)
    orc.set_occupancy(5, 5, True)
    assert_same_structure(gpu, orc.export())


def test_snapshot_roundtrip_and_reference_bytes(rl, oracle_mod):
    g = random_map(20, 14, 0.12, 55)
    gpu = make_gpu(rl, g, 16)
    data = rl.serialize_cddt(gpu)
    back = rl.deserialize_cddt(data)
    assert rl.serialize_cddt(back) == data
    assert_same_structure(back, gpu.export())
    if oracle_mod.ref_available():
        ref = oracle_mod.RefCddt(g, 16)
        assert ref.serialize() == data
        ref.prune()
        pr = rl.deserialize_cddt(ref.serialize())
        assert pr.pruned()
        assert_same_structure(pr, ref.export())
    bad = bytearray(data)
    bad[0] ^= 0xFF
    with pytest.raises(rl.ParseError):
        rl.deserialize_cddt(bytes(bad))
    with pytest.raises(rl.ParseError):
        rl.deserialize_cddt(data[:-3])
    with pytest.raises(rl.ParseError):
        rl.deserialize_cddt(data + b"\0")
    with pytest.raises(rl.ParseError):
        rl.deserialize_cddt(b"")


def test_maze_cfg2_build_and_casts(rl, oracle_mod, synth):
    """Config 2 map (2000x2000 maze, theta_disc 120, max_range 500): structure
    and 200k casts bit-exact with the oracle."""
    import torch
    g = synth.maze_map()
    gpu = make_gpu(rl, g, 120, 500.0)
    orc = oracle_mod.OracleCddt(g, 120, 500.0)
    assert_same_structure(gpu, orc.export())
    qx, qy, qt = synth.free_queries(g, 200_000, seed=21)
    want = orc.cast_batch(qx, qy, qt)
    got = gpu.cast_batch(dev(qx), dev(qy), dev(qt))
    torch.cuda.synchronize()
    assert np.array_equal(host(got), want["out32"])


# ---- full-size pins against hashes produced by the unmodified reference
# (tests/golden/make_golden.py --large; config-3 PCDDT took the reference
# 784 s single-threaded) ----
import hashlib  # noqa: E402
import json  # noqa: E402
from pathlib import Path  # noqa: E402

_LARGE_PATH = Path(__file__).resolve().parent / "golden" / "large.json"
LARGE = json.loads(_LARGE_PATH.read_text()) if _LARGE_PATH.exists() else {}


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _map_for(name, synth):
    if name.startswith("cfg1"):
        return synth.rect_map()
    if name.startswith("cfg3"):
        return synth.polygon_map()
    return synth.maze_map()


@pytest.mark.parametrize("name", ["cfg1_cddt", "cfg1_pcddt", "cfg2_cddt", "cfg3_cddt",
                                  "cfg3_pcddt"])
def test_full_size_structure_and_casts_vs_reference_hashes(rl, synth, name):
    import torch
    want = LARGE.get(name)
    if want is None:
        pytest.skip("tests/golden/large.json missing")
    g = _map_for(name, synth)
    c = make_gpu(rl, g, want["theta_disc"], want["max_range"], prune=want["pruned"])
    e = c.export()
    assert c.zero_point_count() == want["info"]["zero_points"]
    assert c.memory_bytes() == want["info"]["memory_bytes"]
    assert _sha(e["zp"]) == want["zp_sha"]
    assert _sha(e["row_off"]) == want["row_off_sha"]
    assert _sha(e["membership"]) == want["membership_sha"]
    qx, qy, qt = synth.free_queries(g, want["queries"], seed=want["query_seed"])
    out = torch.empty(qx.size, dtype=torch.float64, device="cuda")
    c.cast_batch_f64(*(dev(a.astype(np.float64)) for a in (qx, qy, qt)), out=out)
    o32 = c.cast_batch(dev(qx), dev(qy), dev(qt))
    torch.cuda.synchronize()
    assert _sha(host(out)) == want["casts_sha"]
    assert _sha(host(o32)) == want["casts_f32_sha"]


def test_cfg3_split_pipeline_16M_vs_reference_hashes(rl, synth):
    """The headline path itself: 16M config-3 queries through the split cast
    pipeline (two pipelines of phase 1 / near field / window passes, batches >=
    8M), f32 ranges sha-equal to float(the reference's f64 casts) on the
    reference-built PCDDT; the GPU-built PCDDT serialises to the reference's
    snapshot bytes (sha in oracle/cfg3_pcddt.sha256); f64 ranges (single-kernel
    path) sha-equal to the reference's."""
    import torch
    from pathlib import Path
    want = LARGE.get("cfg3_pcddt_split16M")
    if want is None:
        pytest.skip("tests/golden/large.json has no cfg3_pcddt_split16M")
    g = synth.polygon_map()
    c = make_gpu(rl, g, 200, 1000.0, prune=True)
    ref_sha = (Path(__file__).resolve().parents[1] / "oracle" / "cfg3_pcddt.sha256").read_text()
    assert _sha(np.frombuffer(rl.serialize_cddt(c), np.uint8)) == ref_sha.split()[0]
    qx, qy, qt = synth.free_queries(g, want["queries"], seed=want["query_seed"])
    o32 = c.cast_batch(dev(qx), dev(qy), dev(qt))
    torch.cuda.synchronize()
    assert _sha(host(o32)) == want["casts_f32_sha"]
    out = c.cast_batch_f64(*(dev(a.astype(np.float64)) for a in (qx, qy, qt)))
    assert _sha(host(out)) == want["casts_sha"]
    # the host-pointer pipeline (chunked H2D / cast / D2H) on the same stream
    assert _sha(c.cast_batch(qx, qy, qt)) == want["casts_f32_sha"]


def test_full_size_edit_rounds_vs_reference_hashes(rl, synth):
    """Config 5: 2000x2000 maze, theta_disc 108, rounds of 50 random 3x3
    insert/remove blocks; zero points bit-exact with the reference after every
    round (hashes from the reference's sequential set_occupancy)."""
    rounds = LARGE.get("cfg5_rounds")
    if not rounds:
        pytest.skip("tests/golden/large.json missing")
    g = synth.maze_map()
    c = make_gpu(rl, g, 108, 0.0)
    for rd in rounds:
        xy, occ = synth.block_edits(2000, 2000, 50, seed=rd["seed"])
        c.set_occupancy_batch(xy, occ)
        e = c.export()
        assert c.zero_point_count() == rd["zero_points"]
        assert _sha(e["zp"]) == rd["zp_sha"]
        assert _sha(e["row_off"]) == rd["row_off_sha"]
        assert _sha(e["membership"]) == rd["membership_sha"]


# ---- oracle_cast and lut_build on the GPU ----
def test_exact_cast_vs_reference_oracle(rl, oracle_mod, synth):
    import math
    import torch
    if not oracle_mod.ref_available():
        pytest.skip("reference not compiled")
    g = synth.rect_map(120, 90, 8, seed=5)
    gpu = make_gpu(rl, g, 36, 60.0)
    ref = oracle_mod.RefCddt(g, 36, 60.0)
    rng = np.random.default_rng(11)
    n = 20000
    x, y = rng.uniform(-2, 122, n), rng.uniform(-2, 92, n)
    t = rng.uniform(-7, 13, n)
    # glibc cos/sin of the normalised angle (what RayQuery + oracle_cast use)
    tn = np.array([rl.normalize_angle_2pi(v) for v in t])
    cs = np.array([math.cos(v) for v in tn])
    sn = np.array([math.sin(v) for v in tn])
    want = ref.oracle_batch(x, y, t)
    got = gpu.exact_cast_batch(dev(x), dev(y), dev(t), dev(cs), dev(sn))
    approx = gpu.exact_cast_batch(dev(x), dev(y), dev(t))
    torch.cuda.synchronize()
    assert np.array_equal(host(got).view(np.uint64), want.view(np.uint64))
    # device sincos: within the north-star range tolerance
    d = np.abs(host(approx) - want)
    assert np.all((d <= 1e-3) | (d <= 1e-4 * np.abs(want)))


def test_lut_build_vs_reference(rl, oracle_mod, synth):
    import torch
    if not oracle_mod.ref_available():
        pytest.skip("reference not compiled")
    g = synth.rect_map(64, 48, 5, seed=9)
    for K, mr in ((16, 0.0), (36, 25.0)):
        gpu = make_gpu(rl, g, 36, mr)
        ref = oracle_mod.RefCddt(g, 36, mr)
        got = gpu.lut_build(K)
        torch.cuda.synchronize()
        assert np.array_equal(host(got).view(np.uint16), ref.lut_build(K))


def test_simulate_scans_vs_reference(rl, oracle_mod, synth):
    """simulate_scan (mcl.cpp:144-154) batched: noise-free beams equal the
    reference oracle_cast; the counter-generator noise is N(0, sigma),
    reproducible per (seed, stream_id) and clamped to [0, max_range]."""
    import math
    import torch
    if not oracle_mod.ref_available():
        pytest.skip("reference not compiled")
    g = synth.rect_map(120, 90, 8, seed=5)
    spec = rl.ScanSpec(61, 4.71238898038469)
    rng = np.random.default_rng(12)
    n = 500
    x, y, t = rng.uniform(1, 119, n), rng.uniform(1, 89, n), rng.uniform(-7, 13, n)
    off = np.array([spec.beam_offset(b) for b in range(spec.beam_count)])
    tb = (t[:, None] + off[None, :]).ravel()
    tn = np.array([rl.normalize_angle_2pi(v) for v in tb])
    cs = np.array([math.cos(v) for v in tn])
    sn = np.array([math.sin(v) for v in tn])
    xr, yr = np.repeat(x, spec.beam_count), np.repeat(y, spec.beam_count)
    for mr in (60.0, 25.0):
        gpu = make_gpu(rl, g, 36, 60.0)  # oracle_cast takes max_range per call
        want = oracle_mod.RefCddt(g, 36, mr).oracle_batch(xr, yr, tb).reshape(n, -1)
        clean = gpu.simulate_scans(dev(x), dev(y), dev(t), spec, mr, 0.0, cos_t=dev(cs),
                                   sin_t=dev(sn))
        torch.cuda.synchronize()
        assert np.abs(host(clean) - want).max() <= 1e-9  # the 1e-12 noise floor
    noisy = gpu.simulate_scans(dev(x), dev(y), dev(t), spec, 25.0, 2.0, seed=3)
    again = gpu.simulate_scans(dev(x), dev(y), dev(t), spec, 25.0, 2.0, seed=3)
    other = gpu.simulate_scans(dev(x), dev(y), dev(t), spec, 25.0, 2.0, seed=3, stream_id=1)
    torch.cuda.synchronize()
    nz, cl = host(noisy), want
    assert np.array_equal(nz, host(again)) and not np.array_equal(nz, host(other))
    assert nz.min() >= 0.0 and nz.max() <= 25.0
    inner = (cl > 8.0) & (cl < 17.0)  # far from both clamps
    r = (nz - cl)[inner]
    assert r.size > 2000 and abs(r.mean()) < 0.15 and abs(r.std() - 2.0) < 0.1


# ---- the deferred-walk batch path (f32, >= 4M queries) ----
def _deferred_vs_oracle(rl, oracle_mod, g, K, mr, qx, qy, qt):
    import torch
    assert qx.size >= (1 << 22)  # large enough for the split kernels
    gpu = make_gpu(rl, g, K, mr)
    got = gpu.cast_batch(dev(qx), dev(qy), dev(qt))
    torch.cuda.synchronize()
    want = oracle_mod.OracleCddt(g, K, mr).cast_batch(qx, qy, qt, want_f64=False, want_hit=False,
                                                      want_res=False)["out32"]
    bad = np.flatnonzero(host(got).view(np.uint32) != want.view(np.uint32))
    assert bad.size == 0, (bad[:10], host(got)[bad[:10]], want[bad[:10]])


def test_deferred_path_maze(rl, oracle_mod, synth):
    g = synth.maze_map(1000, 1000, 0.10, 8)
    qx, qy, qt = synth.free_queries(g, 5_000_000, seed=3)
    _deferred_vs_oracle(rl, oracle_mod, g, 120, 500.0, qx, qy, qt)


def test_deferred_path_edge_cases(rl, oracle_mod):
    """Origins anywhere (off-map, occupied, next to walls), a tiny max_range
    (below the near field and the verification window), theta_disc 4, angles
    far outside [0, 2pi)."""
    rng = np.random.default_rng(5)
    g = (rng.random((61, 83)) < 0.25).astype(np.uint8)
    n = 1 << 22
    qx = rng.uniform(-3, 86, n).astype(np.float32)
    qy = rng.uniform(-3, 64, n).astype(np.float32)
    qt = rng.uniform(-40, 40, n).astype(np.float32)
    qx[: n // 8] = np.round(qx[: n // 8])  # exactly on lattice lines
    # exactly on pixel-centre projections: ties between the query's projected
    # x' and stored zero points along the axis-aligned slices
    qx[n // 8: n // 4] = np.round(qx[n // 8: n // 4]) + 0.5
    qy[n // 8: n // 4] = np.round(qy[n // 8: n // 4]) + 0.5
    qt[n // 8: n // 4] = (np.pi / 2) * rng.integers(0, 4, n // 8)
    for K, mr in ((4, 0.0), (24, 0.5), (216, 2.0)):
        _deferred_vs_oracle(rl, oracle_mod, g, K, mr, qx, qy, qt)


def test_deferred_path_equals_single_kernel_cfg3(rl, synth):
    """Config-3 PCDDT: the split f32 batch equals float() of the single-kernel
    f64 batch on 8M queries, and the pipelined host-buffer path (an 8M-query
    body chunk plus the 4M/2M/1M/1M tail ramp, split and single-kernel chunks
    mixed) returns the same ranges."""
    import torch
    g = synth.polygon_map()
    gpu = make_gpu(rl, g, 200, 1000.0, prune=True)
    n = 8_000_000 + (1 << 23) + 12_345
    qx, qy, qt = synth.free_queries(g, n, seed=77)
    split = gpu.cast_batch(dev(qx), dev(qy), dev(qt))
    m = 8_000_000
    whole = gpu.cast_batch_f64(*(dev(a[:m].astype(np.float64)) for a in (qx, qy, qt)))
    torch.cuda.synchronize()
    assert torch.equal(split[:m], whole.float())
    hosted = gpu.cast_batch(qx, qy, qt)
    assert np.array_equal(hosted, host(split))


def test_concurrent_batches_on_two_streams(rl, synth):
    """Two large batches on different streams against one handle (the pattern of
    the pipelined host path) give the same results as one after the other."""
    import torch
    g = synth.maze_map(800, 800, 0.1, 2)
    gpu = make_gpu(rl, g, 120, 300.0)
    a = [dev(v) for v in synth.free_queries(g, 5_000_000, seed=1)]
    b = [dev(v) for v in synth.free_queries(g, 5_000_000, seed=2)]
    ra = gpu.cast_batch(*a)
    rb = gpu.cast_batch(*b)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    oa, ob = torch.empty_like(ra), torch.empty_like(rb)
    for _ in range(3):
        with torch.cuda.stream(s1):
            gpu.cast_batch(*a, out=oa)
        with torch.cuda.stream(s2):
            gpu.cast_batch(*b, out=ob)
    torch.cuda.synchronize()
    assert torch.equal(oa, ra) and torch.equal(ob, rb)


def test_default_stream_ordering(rl, synth):
    """Work queued on torch's default stream before a cast is visible to it:
    the wrappers pass torch's legacy default stream explicitly (a NULL stream
    means the handle's own, unordered stream in the C ABI)."""
    import torch
    from paper_1705_01167_b200 import _lib
    assert torch.cuda.current_stream().cuda_stream == 0
    assert _lib.torch_stream(torch.device("cuda", 0)).value == _lib.CUDA_STREAM_LEGACY
    g = synth.maze_map(800, 800, 0.1, 2)
    gpu = make_gpu(rl, g, 120, 300.0)
    a = [dev(v) for v in synth.free_queries(g, 1_000_000, seed=3)]
    b = [dev(v) for v in synth.free_queries(g, 1_000_000, seed=4)]
    want = gpu.cast_batch(*b)
    torch.cuda.synchronize()
    for _ in range(3):
        q = [t.clone() for t in a]
        torch.cuda._sleep(50_000_000)  # keep the default stream busy (~25 ms)
        for dst, src in zip(q, b):
            dst.copy_(src)  # queued behind the sleep
        got = gpu.cast_batch(*q)
        torch.cuda.synchronize()
        assert torch.equal(got, want)


_QUEUE_CHECK = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import paper_1705_01167_b200 as rl
from paper_1705_01167_b200 import synth
g = synth.polygon_map()
c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(1000.0, 200), prune=True)
q = [torch.from_numpy(a).cuda() for a in synth.free_queries(g, 8_000_000, seed=78)]
split = c.cast_batch(*q)
whole = c.cast_batch_f64(*(t.double() for t in q))
torch.cuda.synchronize()
print("EQUAL" if torch.equal(split, whole.float()) else "DIFFER")
"""


@pytest.mark.parametrize("cap,plan", [("", ""), ("4096", ""), ("1", ""), ("", "full"),
                                      ("1", "full"), ("", "one"), ("", "short-one")])
def test_window_pass_queues(cap, plan):
    """The window passes hand unfinished queries on through bounded queues;
    with the queue capacity forced tiny (RL_CDDT_CONT_CAP) nearly every
    continuation takes the queue-full path, which must give the same answers.
    The batch-size plan is forced too: by default 8M queries run as two
    pipelines with the short window plan {2}; "full" forces caps {1, 2, 4},
    "one" a single pipeline with the full plan, "short-one" a single pipeline
    with the short plan."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    env = dict(os.environ)
    if cap:
        env["RL_CDDT_CONT_CAP"] = cap
    if plan in ("full", "one"):
        env["RL_SHORT_PLAN_MAX"] = "0"
    if plan in ("one", "short-one"):
        env["RL_TWO_PIPE_MIN"] = "1000000000"
    root = str(Path(__file__).resolve().parent.parent)
    r = subprocess.run([sys.executable, "-c", _QUEUE_CHECK.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().endswith("EQUAL"), r.stdout + r.stderr[-2000:]


def test_casts_after_every_structure_change(rl, synth):
    """Queries read derived per-row records (CSR range + search probes) that
    must be rebuilt after edits, prune and snapshot loads: after each change
    the batched casts (split path, >= 4M queries, and the single f64 kernel)
    equal those of a structure built fresh from the same grid."""
    import torch
    g = synth.maze_map(400, 400, 0.10, 6)
    K, mr = 108, 250.0
    q = [dev(a) for a in synth.free_queries(g, 1 << 22, seed=41)]
    q64 = [t.double() for t in q]

    def same(a, b):
        ra, rb = a.cast_batch(*q), b.cast_batch(*q)
        fa, fb = a.cast_batch_f64(*q64), b.cast_batch_f64(*q64)
        torch.cuda.synchronize()
        assert torch.equal(ra, rb) and torch.equal(fa, fb)

    gpu = make_gpu(rl, g, K, mr)
    for rnd in range(3):
        xy, occ = synth.block_edits(400, 400, 60, seed=700 + rnd)
        gpu.set_occupancy_batch(xy, occ)
    edited = gpu.export()["grid"]
    same(gpu, make_gpu(rl, edited, K, mr))
    gpu.prune()
    pruned = make_gpu(rl, edited, K, mr, prune=True)
    same(gpu, pruned)
    same(rl.deserialize_cddt(rl.serialize_cddt(gpu)), pruned)


def test_f64_batch_optional_outputs(rl, synth):
    """Every optional output of rl_cddt_cast_batch_f64 (range, hit cell,
    resolving row/index) may be omitted independently."""
    import itertools
    import torch
    g = synth.rect_map(300, 200, 20, seed=3)
    gpu = make_gpu(rl, g, 72, 150.0)
    q = [dev(a.astype(np.float64)) for a in synth.free_queries(g, 50_000, seed=5)]
    n = q[0].numel()
    full = dict(out=torch.empty(n, dtype=torch.float64, device="cuda"),
                hit=torch.empty(n, dtype=torch.int32, device="cuda"),
                res_row=torch.empty(n, dtype=torch.int64, device="cuda"),
                res_idx=torch.empty(n, dtype=torch.int32, device="cuda"))
    gpu.cast_batch_f64(*q, **full)
    torch.cuda.synchronize()
    for mask in itertools.product((0, 1), repeat=4):
        part = {k: torch.full_like(v, -7) for (k, v), m in zip(full.items(), mask) if m}
        gpu.cast_batch_f64(*q, **{k: part.get(k) for k in full})
        torch.cuda.synchronize()
        for k, v in part.items():
            assert torch.equal(v, full[k]), (mask, k)


@pytest.mark.parametrize("seed", [101, 202, 303])
def test_split_path_random_structures(rl, oracle_mod, synth, seed):
    """Randomised split-path parity: odd map sizes (not multiples of 32),
    random occupancy, theta_disc and max_range, CDDT and PCDDT, 4M+ queries
    from anywhere around the map, bit-exact against the restatement."""
    import torch
    rng = np.random.default_rng(seed)
    w, h = int(rng.integers(37, 300)), int(rng.integers(5, 260))
    g = (rng.random((h, w)) < rng.uniform(0.02, 0.3)).astype(np.uint8)
    K = int(rng.integers(2, 160)) * 2
    mr = float(rng.choice([0.0, rng.uniform(0.5, 4.0), rng.uniform(5.0, 400.0)]))
    prune = bool(seed % 2)
    n = (1 << 22) + int(rng.integers(0, 100_000))
    qx = rng.uniform(-2, w + 2, n).astype(np.float32)
    qy = rng.uniform(-2, h + 2, n).astype(np.float32)
    qt = rng.uniform(-7, 13, n).astype(np.float32)
    gpu = make_gpu(rl, g, K, mr, prune=prune)
    got = gpu.cast_batch(dev(qx), dev(qy), dev(qt))
    torch.cuda.synchronize()
    orc = oracle_mod.OracleCddt(g, K, mr)
    if prune:
        orc.prune()
    want = orc.cast_batch(qx, qy, qt, want_f64=False, want_hit=False, want_res=False)["out32"]
    bad = np.flatnonzero(host(got).view(np.uint32) != want.view(np.uint32))
    assert bad.size == 0, (w, h, K, mr, prune, bad[:10])


_EDIT_PATHS = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r})
import oracle
import paper_1705_01167_b200 as rl
from paper_1705_01167_b200 import synth
K, mr = 108, 250.0
g = synth.maze_map(400, 400, 0.10, 8)
def make(grid):
    return rl.Cddt(rl.OccupancyGrid.from_array(grid), rl.RangeMethodConfig(mr, K))
gpu, orc = make(g), oracle.OracleCddt(g, K, mr)
q = [torch.from_numpy(a).cuda().double() for a in synth.free_queries(g, 200_000, seed=5)]
rng = np.random.default_rng(9)
for rnd in range(14):
    if rnd % 3 == 2:  # a wall of blocks along one grid row: many records for the same rows
        y0 = int(rng.integers(5, 390))
        xs = np.arange(5, 395, 4)
        xy = np.array([(x + dx, y0 + dy) for x in xs for dy in range(3) for dx in range(3)],
                      np.int32)
        occ = np.full(len(xy), 1 if rnd % 2 else 0, np.uint8)
    else:
        xy, occ = synth.block_edits(400, 400, 50, seed=300 + rnd)
    for (x, y), o in zip(xy, occ):
        orc.set_occupancy(int(x), int(y), bool(o))
    gpu.set_occupancy_batch(xy, occ)
    e, o = gpu.export(), orc.export()
    for k in ("zp", "row_off", "membership"):
        if not np.array_equal(np.asarray(e[k]).view(np.uint8), np.asarray(o[k]).view(np.uint8)):
            print("DIFFER", rnd, k); sys.exit(0)
    fresh = make(gpu.export()["grid"])
    a, b = gpu.cast_batch_f64(*q), fresh.cast_batch_f64(*q)
    torch.cuda.synchronize()
    if not torch.equal(a, b):
        print("CASTS DIFFER", rnd); sys.exit(0)
if rl.serialize_cddt(gpu) != rl.serialize_cddt(fresh):
    print("SNAPSHOT DIFFERS"); sys.exit(0)
gpu.prune(); fresh.prune()
e, f = gpu.export(), fresh.export()
if not all(np.array_equal(np.asarray(e[k]), np.asarray(f[k])) for k in ("zp", "row_off")):
    print("PRUNE DIFFERS"); sys.exit(0)
print("EQUAL", gpu.zero_point_count())
"""


@pytest.mark.parametrize("append", ["", "0", "3000"])
def test_edit_paths_in_place_relocated_relayout(append):
    """Edit batches after the first merge the touched rows where they lie,
    move rows that outgrow their slots to the append area, and fall back to a
    full relayout when that area is exhausted (RL_EDIT_APPEND_SLOTS forces
    it: 0 = every batch, 3000 = every few). Every path must leave the zero
    points, offsets and membership bit-identical to the sequential
    restatement, casts equal to a fresh build, and the snapshot and a later
    prune equal to those of the fresh build."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    env = dict(os.environ)
    if append:
        env["RL_EDIT_APPEND_SLOTS"] = append
    root = str(Path(__file__).resolve().parent.parent)
    r = subprocess.run([sys.executable, "-c", _EDIT_PATHS.format(root=root)], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip().split()[0] == "EQUAL", r.stdout + r.stderr[-2000:]


def test_edit_batch_larger_than_a_chunk(rl, oracle_mod):
    """A batch of more than 2^20 edits is replayed in order in chunks (the
    device stamp keeps 20 bits of edit index): the last edit of each cell
    wins across the chunk boundary, and the structure equals a fresh build of
    the final grid (proj/tests/test_cddt.cpp:578-604)."""
    g = random_map(64, 48, 0.2, 21)
    K = 16
    gpu = make_gpu(rl, g, K)
    rng = np.random.default_rng(77)
    n = (1 << 20) + 4099
    xy = np.stack([rng.integers(0, 64, n), rng.integers(0, 48, n)], 1).astype(np.int32)
    occ = rng.integers(0, 2, n).astype(np.uint8)
    # cells whose last edit lies past the chunk boundary and whose earlier ones differ
    xy[-3:] = [[5, 5], [6, 6], [5, 5]]
    xy[:2] = [[5, 5], [6, 6]]
    occ[:2], occ[-3:] = [1, 1], [1, 0, 0]
    final = np.array(g, np.uint8, copy=True)
    final[xy[:, 1], xy[:, 0]] = occ  # numpy keeps the last write per index
    assert final[5, 5] == 0 and final[6, 6] == 0
    gpu.set_occupancy_batch(xy, occ)
    assert np.array_equal(gpu.export()["grid"], final)
    assert_same_structure(gpu, oracle_mod.OracleCddt(final, K).export())


def test_host_path_pageable_pinned_and_mixed(rl, synth):
    """rl_cddt_cast_batch_host with pageable buffers (staged through the pinned
    ring by host threads), pinned buffers (copied directly) and a mix, at sizes
    around the staging chunk (ragged last chunk, fewer chunks than lanes): all
    equal the device-pointer path bit for bit."""
    import torch
    g = synth.rect_map(300, 260, 14, seed=4)
    gpu = make_gpu(rl, g, 108, 200.0)
    nmax = (9 << 20) + 12345
    qx, qy, qt = synth.free_queries(g, nmax, seed=21)
    want = host(gpu.cast_batch(dev(qx), dev(qy), dev(qt)))
    torch.cuda.synchronize()
    pin = [torch.from_numpy(a).pin_memory().numpy() for a in (qx, qy, qt)]
    for n in (nmax, (4 << 20), (1 << 20) + 7, 1000):
        got = gpu.cast_batch(qx[:n], qy[:n], qt[:n])  # pageable in, pageable out
        assert np.array_equal(got.view(np.uint32), want[:n].view(np.uint32)), n
        out = torch.empty(n, dtype=torch.float32).pin_memory().numpy()
        gpu.cast_batch(pin[0][:n], pin[1][:n], pin[2][:n], out=out)  # all pinned
        assert np.array_equal(out.view(np.uint32), want[:n].view(np.uint32)), n
        out2 = np.zeros(n, dtype=np.float32)
        gpu.cast_batch(pin[0][:n], qy[:n], pin[2][:n], out=out2)  # mixed
        assert np.array_equal(out2.view(np.uint32), want[:n].view(np.uint32)), n


def test_cast_queries_host_rayquery_array(rl, oracle_mod, synth):
    """rl_cddt_cast_queries_host: an [n, 3] array of RayQuery rows (doubles, not
    float-representable) from pageable and pinned host memory equals the f64
    device path bit for bit, at sizes around the pipeline's chunks, and the
    reference / restatement on a sample."""
    import torch
    g = synth.rect_map(300, 260, 14, seed=4)
    gpu = make_gpu(rl, g, 108, 200.0)
    nmax = (5 << 20) + 777
    qx, qy, qt = synth.free_queries(g, nmax, seed=23)
    rng = np.random.default_rng(6)
    q = np.stack([qx.astype(np.float64) + rng.uniform(-1e-4, 1e-4, nmax),
                  qy.astype(np.float64) + rng.uniform(-1e-4, 1e-4, nmax),
                  qt.astype(np.float64) * 3.0 - 4.0 + rng.uniform(-1e-6, 1e-6, nmax)], axis=1)
    want = host(gpu.cast_batch_f64(dev(q[:, 0]), dev(q[:, 1]), dev(q[:, 2])))
    torch.cuda.synchronize()
    qp = torch.from_numpy(q).pin_memory().numpy()
    for n in (nmax, 2 << 20, (1 << 19) + 1, 3, 0):
        got = gpu.cast_queries(q[:n])  # pageable in and out
        assert np.array_equal(got.view(np.uint64), want[:n].view(np.uint64)), n
        out = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
        gpu.cast_queries(qp[:n], out=out)  # pinned in and out
        assert np.array_equal(out.view(np.uint64), want[:n].view(np.uint64)), n
        out2 = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
        gpu.cast_queries(q[:n], out=out2)  # pageable in, pinned out
        assert np.array_equal(out2.view(np.uint64), want[:n].view(np.uint64)), n
    m = 20_000
    if oracle_mod.ref_available():
        ref, _ = oracle_mod.RefCddt(g, 108, 200.0).cast_pair_batch(q[:m, 0], q[:m, 1], q[:m, 2])
    else:
        o = oracle_mod.OracleCddt(g, 108, 200.0)
        m = 2_000
        ref = np.array([o.cast(*q[i]) for i in range(m)])
    assert np.array_equal(want[:m].view(np.uint64), np.asarray(ref).view(np.uint64))
    with pytest.raises(ValueError):
        gpu.cast_queries(np.zeros((4, 2)))
