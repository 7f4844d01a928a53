"""GPU parity of the fused beam sensor model (sensor_update, proj/src/mcl.cpp:58-120).

Tolerance (BASELINE.json north_star): particle weights within 1e-5 relative of
the reference. The casts inside are bit-exact (test_gpu_cddt.py), so the only
differences are CUDA vs glibc log/exp/erf rounding and the reduction order of
the normalising sum.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FOV = 4.71238898038469
W_RTOL = 1e-5


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def setup_cfg2(rl, synth, n, seed=9):
    g = synth.maze_map()
    x, y, t = synth.free_pose(g, 10, seed=5)
    px, py, pt = synth.particles(x, y, t, n, 10.0, 0.1, seed=seed)
    scan = synth.scan(g, x, y, t, 61, FOV, 500.0, 8.0, 0.05, seed=13)
    return g, px, py, pt, scan


def test_sensor_analytic_vs_reference(rl, oracle_mod, synth):
    import torch
    g, px, py, pt, scan = setup_cfg2(rl, synth, 500)
    method = rl.make_method("cddt", rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(500.0, 120))
    beam = rl.BeamModelParams(sigma_hit=8.0, z_max=500.0)
    parts = {k: dev(v) for k, v in dict(x=px, y=py, theta=pt, weight=np.zeros_like(px)).items()}
    logw = torch.empty(px.size, dtype=torch.float64, device="cuda")
    ok = rl.sensor_update(parts, method, dev(scan), rl.ScanSpec(61, FOV), beam, logw=logw)
    assert ok
    w = parts["weight"].cpu().numpy()
    assert abs(w.sum() - 1.0) < 1e-9
    p = oracle_mod.beam_params(sigma_hit=8.0, z_max=500.0)
    if oracle_mod.ref_available():
        ref = oracle_mod.RefCddt(g, 120, 500.0)
        want, deg = ref.sensor_update(px, py, pt, scan, FOV, p, paired=False)
        assert not deg
        np.testing.assert_allclose(w, want, rtol=W_RTOL, atol=1e-300)
        # the paired path gives identical answers (proj/tests/test_mcl.cpp:257-283)
        want_p, _ = ref.sensor_update(px, py, pt, scan, FOV, p, paired=True)
        np.testing.assert_allclose(w, want_p, rtol=W_RTOL, atol=1e-300)
    orc = oracle_mod.OracleCddt(g, 120, 500.0)
    lw, wo, deg = orc.sensor_update(px, py, pt, scan, FOV, p)
    np.testing.assert_allclose(logw.cpu().numpy(), lw, rtol=1e-12)
    np.testing.assert_allclose(w, wo, rtol=W_RTOL, atol=1e-300)


def test_sensor_table_vs_oracle(rl, oracle_mod, synth):
    import torch
    g, px, py, pt, scan = setup_cfg2(rl, synth, 2500)
    method = rl.make_method("cddt", rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(500.0, 120))
    beam = rl.BeamModelParams(sigma_hit=8.0, z_max=500.0)
    table = rl.beam_table(beam, 501, 1.0)
    p = oracle_mod.beam_params(sigma_hit=8.0, z_max=500.0)
    # host table equals the restatement's table (both from beam_likelihood)
    ot = np.empty((501, 501), np.float32)
    oracle_mod.orc_lib().orc_beam_table(p.ctypes.data, 501, 1.0, ot.ctypes.data)
    assert np.array_equal(table.view(np.uint32), ot.view(np.uint32))
    parts = {k: dev(v) for k, v in dict(x=px, y=py, theta=pt, weight=np.zeros_like(px)).items()}
    logw = torch.empty(px.size, dtype=torch.float64, device="cuda")
    assert rl.sensor_update(parts, method, dev(scan), rl.ScanSpec(61, FOV), beam, table=dev(table),
                            logw=logw)
    lw, wo, _ = oracle_mod.OracleCddt(g, 120, 500.0).sensor_update(px, py, pt, scan, FOV, p,
                                                                    table=table)
    np.testing.assert_allclose(logw.cpu().numpy(), lw, rtol=1e-12)
    np.testing.assert_allclose(parts["weight"].cpu().numpy(), wo, rtol=W_RTOL, atol=1e-300)


def test_sensor_degenerate_reset(rl, synth):
    # proj/tests/test_mcl.cpp:285-305: all likelihoods underflow -> uniform, False
    import torch
    g = synth.maze_map(400, 400, 0.1, 3)
    method = rl.make_method("cddt", rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(100.0, 24))
    n = 64
    parts = dict(x=torch.full((n,), 200.5, dtype=torch.float64, device="cuda"),
                 y=torch.full((n,), 200.5, dtype=torch.float64, device="cuda"),
                 theta=torch.zeros(n, dtype=torch.float64, device="cuda"),
                 weight=torch.zeros(n, dtype=torch.float64, device="cuda"))
    beam = rl.BeamModelParams(w_hit=1.0, w_short=0.0, w_max=0.0, w_rand=0.0, sigma_hit=0.01,
                              z_max=100.0)
    scan = torch.zeros(61, dtype=torch.float64, device="cuda")
    parts["x"][:] = 10_000.0  # off-map: every cast reads max_range, hit density underflows
    ok = rl.sensor_update(parts, method, scan, rl.ScanSpec(61, FOV), beam)
    assert not ok
    np.testing.assert_allclose(parts["weight"].cpu().numpy(), 1.0 / n)


def test_scan_length_mismatch(rl, synth):
    import torch
    g = synth.maze_map(200, 200, 0.1, 3)
    method = rl.make_method("cddt", rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(100.0, 24))
    parts = {k: torch.zeros(4, dtype=torch.float64, device="cuda") for k in ("x", "y", "theta",
                                                                            "weight")}
    with pytest.raises(ValueError):
        rl.sensor_update(parts, method, torch.zeros(60, dtype=torch.float64, device="cuda"),
                         rl.ScanSpec(61, FOV), rl.BeamModelParams(z_max=100.0))


@pytest.mark.parametrize("table_model", [True, False])
def test_sensor_logw_chunking_invariant(rl, oracle_mod, synth, table_model):
    """A particle's log-weight does not depend on the batch it is scored in:
    one 40k-particle call equals five 8k calls bit for bit, and matches the
    restatement."""
    import torch
    from paper_1705_01167_b200 import _lib
    n = 40_000
    g, px, py, pt, scan = setup_cfg2(rl, synth, n, seed=21)
    method = rl.make_method("cddt", rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(500.0, 120))
    beam = rl.BeamModelParams(sigma_hit=8.0, z_max=500.0)
    table = dev(rl.beam_table(beam, 501, 1.0)) if table_model else None
    bp = beam.c()
    gx, gy, gt, gs = dev(px), dev(py), dev(pt), dev(scan)

    def logw(lo, hi):
        out = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
        _lib.check(_lib.lib().rl_sensor_logw(
            method.cddt.handle, gx[lo:].data_ptr(), gy[lo:].data_ptr(), gt[lo:].data_ptr(),
            hi - lo, gs.data_ptr(), 61, FOV, _lib.C.byref(bp),
            table.data_ptr() if table is not None else None, 501, 1.0, out.data_ptr(), None))
        return out.cpu().numpy()

    full = logw(0, n)
    parts = np.concatenate([logw(lo, min(n, lo + 8000)) for lo in range(0, n, 8000)])
    np.testing.assert_array_equal(full, parts)
    p = oracle_mod.beam_params(sigma_hit=8.0, z_max=500.0)
    lw, _, _ = oracle_mod.OracleCddt(g, 120, 500.0).sensor_update(
        px[:4000], py[:4000], pt[:4000], scan, FOV, p,
        table=table.cpu().numpy() if table is not None else None)
    np.testing.assert_allclose(full[:4000], lw, rtol=1e-12)


def test_paired_beams_bitwise(rl, tmp_path):
    """The paired-beam sensor kernel (one row search per opposite-direction
    beam pair, mcl.cpp:66-96) gives byte-identical log-weights to one cast per
    beam: on maze and rectangle maps, headings on and between direction-lattice
    points (pairs that are not exactly opposite fall back to two casts),
    occupied and off-map origins, non-clear origins (near-field walks), and
    scans of 1, 2 (fov pi), 7, 40, 61, 90 (fov 2 pi) and 121 beams."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    here = Path(__file__).resolve().parent
    outs = {}
    for paired in ("1", "0"):
        out = tmp_path / f"p{paired}.npz"
        env = dict(os.environ, RL_SENSOR_PAIRED=paired)
        r = subprocess.run([sys.executable, str(here / "sensor_pair_probe.py"), str(out)], env=env,
                           capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        outs[paired] = np.load(out)
    a, b = outs["1"], outs["0"]
    assert sorted(a.files) == sorted(b.files) and len(a.files) == 42
    for k in a.files:
        assert a[k].tobytes() == b[k].tobytes(), k
