"""Config-4 particle-filter update timing (40k particles x 61 beams), for
profiling: python scripts/pf_timing.py [iterations]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402

it = int(sys.argv[1]) if len(sys.argv) > 1 else 50
print(bench.pf_update_timing(it, 0))
