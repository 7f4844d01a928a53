
import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import oracle
import paper_1705_01167_b200 as rl
from paper_1705_01167_b200 import synth
K, mr = 108, 250.0
g = synth.maze_map(400, 400, 0.10, 8)
def make(grid):
    return rl.Cddt(rl.OccupancyGrid.from_array(grid), rl.RangeMethodConfig(mr, K))
gpu, orc = make(g), oracle.OracleCddt(g, K, mr)
q = [torch.from_numpy(a).cuda().double() for a in synth.free_queries(g, 200_000, seed=5)]
rng = np.random.default_rng(9)
for rnd in range(14):
    if rnd % 3 == 2:  # a wall of blocks along one grid row: many records for the same rows
        y0 = int(rng.integers(5, 390))
        xs = np.arange(5, 395, 4)
        xy = np.array([(x + dx, y0 + dy) for x in xs for dy in range(3) for dx in range(3)],
                      np.int32)
        occ = np.full(len(xy), 1 if rnd % 2 else 0, np.uint8)
    else:
        xy, occ = synth.block_edits(400, 400, 50, seed=300 + rnd)
    for (x, y), o in zip(xy, occ):
        orc.set_occupancy(int(x), int(y), bool(o))
    gpu.set_occupancy_batch(xy, occ)
    e, o = gpu.export(), orc.export()
    for k in ("zp", "row_off", "membership"):
        if not np.array_equal(np.asarray(e[k]).view(np.uint8), np.asarray(o[k]).view(np.uint8)):
            print("DIFFER", rnd, k); sys.exit(0)
    fresh = make(gpu.export()["grid"])
    a, b = gpu.cast_batch_f64(*q), fresh.cast_batch_f64(*q)
    torch.cuda.synchronize()
    if not torch.equal(a, b):
        print("CASTS DIFFER", rnd); sys.exit(0)
if rl.serialize_cddt(gpu) != rl.serialize_cddt(fresh):
    print("SNAPSHOT DIFFERS"); sys.exit(0)
gpu.prune(); fresh.prune()
e, f = gpu.export(), fresh.export()
if not all(np.array_equal(np.asarray(e[k]), np.asarray(f[k])) for k in ("zp", "row_off")):
    print("PRUNE DIFFERS"); sys.exit(0)
print("EQUAL", gpu.zero_point_count())
