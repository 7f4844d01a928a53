"""Golden digests of the reference's casts of 16M config-3 queries on the
reference-built PCDDT (oracle/_ref/cfg3_pcddt.rlc from scripts/make_ref_pcddt.py,
loaded through its own deserialize_cddt), for the GPU's split cast pipeline
(batches >= 8M queries run as two pipelines of phase 1 / near field / window
passes). Written into tests/golden/large.json as "cfg3_pcddt_split16M".

    python tests/golden/make_cfg3_split_golden.py
"""
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_1705_01167_b200 import synth  # noqa: E402

if __name__ == "__main__":
    oracle.build(ref=True)
    blob = (ROOT / "oracle" / "_ref" / "cfg3_pcddt.rlc").read_bytes()
    want = (ROOT / "oracle" / "cfg3_pcddt.sha256").read_text().split()[0]
    assert hashlib.sha256(blob).hexdigest() == want
    ref = oracle.RefCddt.deserialize(blob)
    g = synth.polygon_map()
    n = 16_000_000
    qx, qy, qt = synth.free_queries(g, n, seed=7)
    r = ref.cast_batch(qx, qy, qt, want_res=False, threads=8)["out64"]
    lj = ROOT / "tests" / "golden" / "large.json"
    large = json.loads(lj.read_text())
    large["cfg3_pcddt_split16M"] = dict(
        queries=n, query_seed=7, structure_sha256=want,
        casts_sha=hashlib.sha256(r.tobytes()).hexdigest(),
        casts_f32_sha=hashlib.sha256(r.astype(np.float32).tobytes()).hexdigest(),
        max_range_hits=int((r == 1000.0).sum()), zeros=int((r == 0.0).sum()))
    lj.write_text(json.dumps(large, indent=1))
    print(large["cfg3_pcddt_split16M"])
