"""bench.py's reference arm on CPU: one JSON line with the driver's keys, the
reference's own CDDT and ray-marching timings, and zero host<->device bytes
(bench.py --impl reference; the GPU arm is exercised on the B200)."""
import json
import subprocess
import sys

import pytest

from conftest import ROOT


def test_reference_arm_json_line(ref_available):
    if not ref_available:
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3", "--ref-sample", "20000", "--rm-sample", "2000"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["warmup"] >= 3
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["ray_march"]["value"] > 0
    assert d["config"]["workload"].startswith("BASELINE config 3")
