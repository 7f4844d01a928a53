"""CPU: the walker's reciprocal-based division (cddt_device.cuh div_rn) equals
IEEE division bit for bit on the walker's operand distribution. FP64
multiply and FMA are IEEE-exact on both the host and sm_100a, so this host
check proves the device sequence."""
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent


def test_fast_division_matches_ieee(tmp_path):
    exe = tmp_path / "fdc"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe), str(HERE / "fast_div_check.c"),
                    "-lm"], check=True)
    r = subprocess.run([str(exe), "1500"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    assert "mismatches 0" in r.stdout
