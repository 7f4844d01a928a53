"""The device normalize_angle_2pi (cddt_device.cuh) skips fmod on [-2pi, 4pi);
check it equals the reference's fmod form (raycast.hpp:20-25) bit for bit on
~1.2 G angles, including values within rounding of the boundaries."""
import shutil
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent


def test_normalize_fast_paths(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = tmp_path / "normalize_check"
    subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false",
                    "-std=c++17", "--expt-relaxed-constexpr", "-o", str(exe),
                    str(ROOT / "normalize_check.cu")], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mismatches: 0 of" in r.stdout
