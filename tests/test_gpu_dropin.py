"""GPU: the reference's own code (Cddt, sensor_update, Mcl; compiled unmodified
into oracle/_ref/dropin_check) driven with the GPU RangeMethod adapter
(include/rl_cddt_rangemethod.hpp) gives bit-identical casts, weights and
closed-loop estimates to the reference's CPU CDDT, a std::vector<RayQuery> through
cast_many equals its cast loop; and the reference's release
gate (proj/tests/test_acceptance.cpp) criteria 2, 3, 4, 9 and 10 pass through
the GPU path (one DROPIN line each)."""
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

EXE = Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "dropin_check"


def test_reference_code_with_gpu_method(rl, oracle_mod):
    if not EXE.exists():
        pytest.skip("oracle/_ref/dropin_check not built (needs the reference sources)")
    r = subprocess.run([str(EXE)], capture_output=True, text=True, timeout=1200)
    print(r.stdout)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("DROPIN")]
    assert len(lines) == 10, r.stdout + r.stderr
    assert r.returncode == 0 and all(" PASS " in ln for ln in lines), r.stdout + r.stderr
