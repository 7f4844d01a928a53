"""Config-3 end-to-end timing through the host-pointer C ABI (pinned host
buffers, H2D + casts + D2H): python scripts/e2e_timing.py"""
import hashlib
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1705_01167_b200 as rl  # noqa: E402

n = int(os.environ.get("NQ", 100_000_000))
g, qx, qy, qt, _ = bench.make_workload(n, 0)
c = rl.Cddt(rl.OccupancyGrid.from_array(g), rl.RangeMethodConfig(1000.0, 200), prune=True)
hx, hy, ht = qx.numpy(), qy.numpy(), qt.numpy()
ho = torch.empty(n, dtype=torch.float32).pin_memory().numpy()
c.cast_batch(hx, hy, ht, out=ho)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    c.cast_batch(hx, hy, ht, out=ho)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print({"lib": os.environ.get("RL_CDDT_LIB", "default"), "ramp": os.environ.get("RL_HOST_RAMP", "default"),
       "ms": ms, "gcasts_per_s": n / ms / 1e6, "sha": hashlib.sha256(ho.tobytes()).hexdigest()[:16]})
