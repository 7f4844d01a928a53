"""Build the config-3 PCDDT with the UNMODIFIED reference (oracle/_ref) and
write its own snapshot format (serialize_cddt, proj/src/cddt.cpp:458-500) to
oracle/_ref/cfg3_pcddt.rlc. Test/baseline infrastructure: the reference's
single-threaded prune of this map takes ~13 minutes, too long for a bench run,
so `bench.py --impl reference` and the config-3 golden casts load this file
through the reference's own deserialize_cddt (cddt.cpp:502-579).
The file is git-ignored but not gpurun-ignored, so it travels to the GPU box
like the .so files.

    python scripts/make_ref_pcddt.py
"""
import hashlib
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_1705_01167_b200 import synth  # noqa: E402

OUT = ROOT / "oracle" / "_ref" / "cfg3_pcddt.rlc"

if __name__ == "__main__":
    oracle.build(ref=True)
    g = synth.polygon_map()
    t0 = time.time()
    ref = oracle.RefCddt(g, 200, 1000.0, prune=True)
    blob = ref.serialize()
    OUT.write_bytes(blob)
    print(f"{OUT} {len(blob)} bytes sha256={hashlib.sha256(blob).hexdigest()} "
          f"build+prune {time.time() - t0:.1f}s", flush=True)
