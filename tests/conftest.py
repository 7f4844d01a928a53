import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def oracle_mod():
    import oracle
    oracle.build(ref=True)
    return oracle


@pytest.fixture(scope="session")
def ref_available(oracle_mod):
    return oracle_mod.ref_available()


@pytest.fixture(scope="session")
def rl():
    """The product package with its CUDA library built and a device present."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    from paper_1705_01167_b200 import build
    build.build_all()
    import paper_1705_01167_b200 as rl
    return rl


@pytest.fixture(scope="session")
def synth():
    from paper_1705_01167_b200 import synth
    return synth


@pytest.fixture(autouse=True)
def _device_bounds_checks(request):
    """With a checked library (built with -DRL_CHECKED and selected through
    RL_CDDT_LIB; the compute-sanitizer stand-in), every GPU test ends with
    zero failed device bounds assertions."""
    yield
    if "gpu" not in request.keywords or not os.environ.get("RL_CHECKED_SUITE"):
        return
    import ctypes as C

    from paper_1705_01167_b200 import _lib
    if _lib._lib is None:
        return
    n, code = C.c_uint64(), C.c_uint32()
    assert _lib._lib.rl_debug_checks(0, C.byref(n), C.byref(code)) == 0
    assert code.value != 0xFFFFFFFF, "RL_CHECKED_SUITE set but the library is not a checked build"
    assert n.value == 0, f"{n.value} device bounds assertions failed (first: site {code.value})"
