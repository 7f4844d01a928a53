"""GPU: the algorithmic sectors per query behind bench.py's roofline
(profiles/sectors.json) equal the instrumented restatement's count on the
bench's own workload: the config-3 PCDDT built on the GPU and the first
`sample` queries of the bench stream. RL_WRITE_SECTORS=1 rewrites the file.
bench.py reads the committed figure; only this test runs the restatement."""
import json
import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SECTORS = ROOT / "profiles" / "sectors.json"


def test_sectors_per_query_fixture(rl, oracle_mod):
    import bench
    sample = 200_000
    g, qx, qy, qt, _ = bench.make_workload(sample, 0)
    c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(1000.0, 200), prune=True)
    orc = oracle_mod.OracleCddt(g, 200, 1000.0, csr=dict(c.export(), pruned=True))
    sec = orc.cast_batch(qx.numpy(), qy.numpy(), qt.numpy(), want_f64=False, want_hit=False,
                         want_res=False, want_sectors=True)["sectors"]
    s_bar = float(np.mean(sec))
    want = {"workload": bench.WORKLOAD["workload"], "query_seed": 7, "sample": sample,
            "sectors_per_query": s_bar,
            "definition": "mean distinct 32-byte sectors the reference algorithm touches per query "
                          "under the reference layout (oracle/cddt_oracle.c), counted by "
                          "tests/test_gpu_sectors.py"}
    if os.environ.get("RL_WRITE_SECTORS"):
        out = ROOT / "gpurun_out" / "sectors.json"
        out.parent.mkdir(exist_ok=True)
        out.write_text(json.dumps(want, indent=1))
    have = json.loads(SECTORS.read_text())
    assert have["sample"] == sample and have["query_seed"] == 7
    assert have["sectors_per_query"] == pytest.approx(s_bar, rel=1e-12)
