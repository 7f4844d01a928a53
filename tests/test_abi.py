"""CPU: the C-ABI library builds for sm_100a, loads without a GPU, and exports
every entry point include/rl_cddt.h declares (no compute calls here)."""
import ctypes
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "rl_cddt.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(rl_\w+)\s*\(", text, re.M)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ("rl_cddt_create", "rl_cddt_cast_batch", "rl_cddt_prune", "rl_cddt_set_occupancy",
              "rl_sensor_update", "rl_last_error"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    from paper_1705_01167_b200 import build
    lib_path = build.build_cuda()
    lib = ctypes.CDLL(str(lib_path))
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_sass_is_sm100a():
    import subprocess
    from paper_1705_01167_b200 import build
    lib_path = build.build_cuda()
    r = subprocess.run(["cuobjdump", "--list-elf", str(lib_path)], capture_output=True, text=True)
    assert "sm_100a" in r.stdout


def test_python_binding_signatures_match_header():
    from paper_1705_01167_b200 import _lib
    lib = _lib.lib()
    assert set(_lib._SIG) == set(declared_symbols())
    assert lib.rl_last_error() is not None


def test_host_errors_without_gpu():
    """Argument validation happens before any device work (invalid_argument)."""
    import paper_1705_01167_b200 as rl
    import pytest
    g = rl.OccupancyGrid(4, 4)
    with pytest.raises(ValueError):
        rl.Cddt(g, rl.RangeMethodConfig(0.0, 7))
    with pytest.raises(ValueError):
        rl.Cddt(g, rl.RangeMethodConfig(-1.0, 8))
    with pytest.raises(ValueError):
        rl.method_kind_from_name("nope")
