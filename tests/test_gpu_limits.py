"""GPU: size limits of the batched path and of the structure, by size-independent
properties and against the restatement/reference.

* A batch of 2^28 + 2^20 queries (above the 2^28-query chunk limit of the split
  pipeline, ~4.3 GB of queries and results) equals the same queries cast in
  4M-query batches, and a strided sample equals the reference.
* A fine direction lattice (theta_disc 2048) builds bit-exactly and casts
  bit-exactly against the restatement, split and monolithic paths.
* Maps whose width is not a multiple of the 32-cell occupancy words, a 1-row
  map and a 1-column map.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.timeout(900)
def test_batch_above_chunk_limit_equals_small_batches(rl, oracle_mod, synth):
    import torch
    g = synth.rect_map()
    c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(300.0, 108))
    n = (1 << 28) + (1 << 20)
    gd = torch.from_numpy(g).cuda()
    qx, qy, qt = synth.free_queries_gpu(gd, 500, 500, n, seed=11)
    big = c.cast_batch(qx, qy, qt)
    ref = torch.empty_like(big)
    step = 1 << 22
    for a in range(0, n, step):
        b = min(n, a + step)
        c.cast_batch(qx[a:b], qy[a:b], qt[a:b], out=ref[a:b])
    torch.cuda.synchronize()
    assert torch.equal(big, ref)
    # a strided sample (including both sides of the 2^28 boundary) against the reference
    idx = np.concatenate([np.arange(0, n, 4099), np.arange((1 << 28) - 5000, (1 << 28) + 5000)])
    sx, sy, st = (t[torch.from_numpy(idx).cuda()].cpu().numpy() for t in (qx, qy, qt))
    want = oracle_mod.OracleCddt(g, 108, 300.0).cast_batch(sx, sy, st, want_f64=False,
                                                           want_hit=False, want_res=False)
    assert np.array_equal(big[torch.from_numpy(idx).cuda()].cpu().numpy(), want["out32"])


def test_fine_direction_lattice(rl, oracle_mod, synth):
    import torch
    g = synth.rect_map(128, 128, 10, seed=21)
    K = 2048
    c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(0.0, K))
    o = oracle_mod.OracleCddt(g, K, 0.0)
    e, oe = c.export(), o.export()
    assert np.array_equal(e["row_off"], oe["row_off"])
    assert np.array_equal(e["zp"].view(np.uint32), oe["zp"].view(np.uint32))
    qx, qy, qt = synth.free_queries(g, 1 << 22, seed=3)  # split path
    got = c.cast_batch(dev(qx), dev(qy), dev(qt))
    torch.cuda.synchronize()
    want = o.cast_batch(qx, qy, qt, want_f64=False, want_hit=False, want_res=False)["out32"]
    assert np.array_equal(got.cpu().numpy(), want)
    got = c.cast_batch(dev(qx[:50000]), dev(qy[:50000]), dev(qt[:50000]))  # monolithic path
    assert np.array_equal(got.cpu().numpy(), want[:50000])


@pytest.mark.parametrize("shape", [(33, 70), (1, 257), (300, 1), (65, 65)])
def test_degenerate_and_ragged_maps(rl, oracle_mod, shape):
    import torch
    h, w = shape
    rng = np.random.default_rng(h * 1000 + w)
    g = (rng.random((h, w)) < 0.15).astype(np.uint8)
    c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(0.0, 36))
    o = oracle_mod.OracleCddt(g, 36, 0.0)
    assert np.array_equal(c.export()["zp"].view(np.uint32), o.export()["zp"].view(np.uint32))
    n = 1 << 22
    qx = rng.uniform(-2, w + 2, n).astype(np.float32)
    qy = rng.uniform(-2, h + 2, n).astype(np.float32)
    qt = rng.uniform(-7, 14, n).astype(np.float32)
    got = c.cast_batch(dev(qx), dev(qy), dev(qt))
    torch.cuda.synchronize()
    want = o.cast_batch(qx, qy, qt, want_f64=False, want_hit=False, want_res=False)["out32"]
    assert np.array_equal(got.cpu().numpy(), want)
    for prune in (True,):
        p = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(0.0, 36), prune=prune)
        o.prune()
        assert np.array_equal(p.export()["zp"].view(np.uint32), o.export()["zp"].view(np.uint32))


def test_f64_batch_above_split_threshold_keeps_double_queries(rl, oracle_mod, synth):
    """A >= 4M f64 batch with range output only must not go through the split
    pipeline (its records hold the query as floats): genuinely double
    coordinates give the same bits as the single-kernel path with hit cells,
    and as the reference / restatement on a sample."""
    import torch
    g = synth.rect_map(300, 260, 14, seed=4)
    c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(200.0, 108))
    n = (1 << 22) + 4097
    qx, qy, qt = synth.free_queries(g, n, seed=33)
    rng = np.random.default_rng(5)
    x = qx.astype(np.float64) + rng.uniform(-1e-4, 1e-4, n)  # not float-representable
    y = qy.astype(np.float64) + rng.uniform(-1e-4, 1e-4, n)
    t = qt.astype(np.float64) + rng.uniform(-1e-6, 1e-6, n)
    dx, dy, dt = (torch.from_numpy(a).cuda() for a in (x, y, t))
    a = c.cast_batch_f64(dx, dy, dt)
    hit = torch.empty(n, dtype=torch.int32, device="cuda")
    b = c.cast_batch_f64(dx, dy, dt, hit=hit)
    torch.cuda.synchronize()
    a, b = a.cpu().numpy(), b.cpu().numpy()
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    m = 20_000
    if oracle_mod.ref_available():
        want, _ = oracle_mod.RefCddt(g, 108, 200.0).cast_pair_batch(x[:m], y[:m], t[:m])
    else:
        o = oracle_mod.OracleCddt(g, 108, 200.0)
        m = 2_000
        want = np.array([o.cast(x[i], y[i], t[i]) for i in range(m)])
    assert np.array_equal(a[:m].view(np.uint64), np.asarray(want).view(np.uint64))
