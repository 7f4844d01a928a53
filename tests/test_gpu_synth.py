"""GPU: the device twin of the query generator (csrc/synth_gpu.cu, used by
bench.py) produces the same bits as the host generator (csrc/synth.c)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("which", ["rect", "polygon"])
def test_gpu_query_generator_matches_host(rl, synth, which):
    import torch
    g = synth.rect_map() if which == "rect" else synth.polygon_map()
    h, w = g.shape
    n, start = 300_000, 12345
    want = synth.free_queries(g, n, seed=7, start=start)
    got = synth.free_queries_gpu(torch.from_numpy(g).cuda(), w, h, n, seed=7, start=start)
    torch.cuda.synchronize()
    for a, b in zip(got, want):
        assert np.array_equal(a.cpu().numpy().view(np.uint32), b.view(np.uint32))
