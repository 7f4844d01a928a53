"""CPU: the walker's reciprocal-based division (cddt_device.cuh div_rn) equals
IEEE division bit for bit on the walker's operand distribution (float and f64
origins). The two-step form is correct by Markstein's theorem (the comment at
div_rn); this is the empirical cross-check. FP64 multiply and FMA are
IEEE-exact on both the host and sm_100a, so the host sequence is the device
sequence."""
import subprocess
from pathlib import Path

HERE = Path(__file__).resolve().parent


def test_fast_division_matches_ieee(tmp_path):
    exe = tmp_path / "fdc"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe), str(HERE / "fast_div_check.c"),
                    "-lm"], check=True)
    r = subprocess.run([str(exe), "1500"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
    import re
    m = re.search(r"checked (\d+) mismatches (\d+)", r.stdout)
    assert m and int(m.group(1)) > 10**8 and m.group(2) == "0", r.stdout
