"""CLI (paper_1705_01167_b200/cli.py): PGM I/O, the reference benchmark query
streams and map id (CPU), and the GPU subcommands against the reference's own
run_random_benchmark / run_grid_benchmark checksums (GPU)."""
import io
import json

import numpy as np
import pytest

from paper_1705_01167_b200 import cli, synth
import paper_1705_01167_b200.rangelib as rl


def test_pgm_round_trip_and_errors(tmp_path):
    g = rl.OccupancyGrid.from_array(synth.rect_map(37, 21, 3, seed=4))
    p = tmp_path / "m.pgm"
    cli.save_pgm(g, str(p))
    assert cli.load_pgm(str(p)) == g
    # P2 with comments (proj/src/grid.cpp:49-108: '#' comments between tokens)
    (tmp_path / "a.pgm").write_text("P2\n# c\n3 2\n# c2\n255\n0 255 127\n128 0 255\n")
    a = cli.load_pgm(str(tmp_path / "a.pgm"))
    assert a.cells.tolist() == [[1, 0, 1], [0, 1, 0]]
    for bad in (b"P3\n1 1\n255\n0", b"P2\n0 1\n255\n", b"P2\n1 1\n300\n0", b"P5\n2 2\n255\n\x00"):
        (tmp_path / "b.pgm").write_bytes(bad)
        with pytest.raises(rl.ParseError):
            cli.load_pgm(str(tmp_path / "b.pgm"))


def test_benchmark_streams_and_map_id_match_reference(oracle_mod):
    if not oracle_mod.ref_available():
        pytest.skip("reference not compiled")
    g = synth.rect_map(120, 90, 8, seed=5)
    grid = rl.OccupancyGrid.from_array(g)
    ref = oracle_mod.RefCddt(g, 36, 0.0)
    orc = oracle_mod.OracleCddt(g, 36, 0.0)
    for random_mode in (True, False):
        n, checksum, mid = ref.bench(random_mode, 4000, 3, stride=7)
        assert mid == cli.map_content_id(grid)
        x, y, t = (cli.random_queries(grid, 4000, 3) if random_mode
                   else cli.grid_queries(grid, 36, 7))
        assert x.size == n
        got = np.array([orc.cast(a, b, c) for a, b, c in zip(x, y, t)])
        assert np.cumsum(got)[-1] == pytest.approx(checksum, rel=1e-12)


@pytest.mark.gpu
def test_cli_gpu_subcommands(rl, oracle_mod, tmp_path, capsys):
    g = synth.maze_map(300, 260, 0.1, 6)
    p = tmp_path / "maze.pgm"
    cli.save_pgm(rl.OccupancyGrid.from_array(g), str(p))
    assert cli.main(["bench", "--map", str(p), "--method", "cddt,pcddt", "--mode", "random",
                     "--queries", "300000", "--theta-disc", "72", "--seed", "5",
                     "--format", "jsonl"]) == 0
    reps = [json.loads(line) for line in capsys.readouterr().out.splitlines()]
    assert [r["method"] for r in reps] == ["cddt-gpu", "pcddt-gpu"]
    if oracle_mod.ref_available():
        n, checksum, mid = oracle_mod.RefCddt(g, 72, 0.0).bench(True, 300000, 5)
        assert reps[0]["queries"] == n and reps[0]["map_id"] == mid
        assert reps[0]["checksum"] == pytest.approx(checksum, rel=1e-12)
    assert cli.main(["cast", "--map", str(p), "-x", "150.5", "-y", "100.5", "--theta", "0.3",
                     "--theta-disc", "72"]) == 0
    r = float(capsys.readouterr().out)
    want = oracle_mod.OracleCddt(g, 72, 0.0).cast(150.5, 100.5, 0.3)
    assert r == want
    assert cli.main(["info", "--map", str(p), "--theta-disc", "72"]) == 0
    assert "pcddt-gpu" in capsys.readouterr().out
    assert cli.main(["mcl-demo", "--map", str(p), "--particles", "2000", "--steps", "40",
                     "--theta-disc", "72", "--out", str(tmp_path / "demo.csv")]) == 0
    res = json.loads(capsys.readouterr().out)
    assert res["median_error"] < 5.0
    assert (tmp_path / "demo.csv").read_text().count("\n") == 41
