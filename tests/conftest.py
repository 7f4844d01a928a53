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
