"""GPU: the scattered-read diagnostic (rl_diag_gather) behind bench.py's
gather ceiling runs, issues the requested reads and sees L2 beat HBM."""
import pytest

pytestmark = pytest.mark.gpu


def test_gather_ceiling(rl):
    import bench
    g = bench.gather_ceiling(0)
    assert set(g) >= {"l2_16MB", "l2_111MB", "hbm_4GB"}
    assert all(v > 1.0 for v in g.values())  # G sectors/s
    assert g["l2_16MB"] > g["hbm_4GB"]


def test_gather_rejects_bad_arguments(rl):
    import ctypes as C

    from paper_1705_01167_b200._lib import RL_EINVAL, lib
    ms, issued = C.c_double(), C.c_uint64()
    assert lib().rl_diag_gather(None, 1 << 20, 1000, None, C.byref(ms), C.byref(issued)) == RL_EINVAL
