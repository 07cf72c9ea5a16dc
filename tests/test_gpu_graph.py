"""Device KNN graph (xknn_graph_bruteforce) vs build_graph_bruteforce: bit-exact neighbour lists
(self first, fp32 ascending-d scores, ties to the lower index), including exact ties and
near-duplicates that defeat the bf16 candidate pass (the certificate's exact fallback)."""
import numpy as np
import pytest

import oracle_lib as O
from gpu_util import torch_cuda

pytestmark = pytest.mark.gpu


def _normalized(w):
    rc, wn, _, _ = O.l2_normalize(w)
    assert rc == 0
    return wn


def _device_graph(wn, k, kprime=0):
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    g, unc = X.graph_bruteforce(torch.from_numpy(wn).cuda(), k, kprime)
    return g.cpu().numpy().view(np.uint32), unc


@pytest.mark.parametrize("n,k", [(1500, 10), (2500, 1), (3000, 33)])
def test_graph_random_full(n, k):
    wn = _normalized(np.random.default_rng(n).standard_normal((n, 512)).astype(np.float32))
    got, _ = _device_graph(wn, k)
    rc, want = O.bruteforce_graph("oracle", wn, k)
    assert rc == 0 and np.array_equal(got, want)


def test_graph_ties_and_near_duplicates():
    rng = np.random.default_rng(5)
    base = rng.standard_normal((300, 512)).astype(np.float32)
    w = np.concatenate([base, base, base + 1e-4 * rng.standard_normal((300, 512)).astype(np.float32),
                        rng.standard_normal((700, 512)).astype(np.float32)])
    wn = _normalized(w)
    got, unc = _device_graph(wn, 8)
    rc, want = O.bruteforce_graph("oracle", wn, 8)
    assert rc == 0 and np.array_equal(got, want)


def test_graph_small_dim_exact_path():
    wn = _normalized(np.random.default_rng(2).standard_normal((400, 64)).astype(np.float32))
    got, _ = _device_graph(wn, 5)
    rc, want = O.bruteforce_graph("oracle", wn, 5)
    assert rc == 0 and np.array_equal(got, want)


def test_graph_large_sampled_rows():
    n, k = 60_000, 20
    wn = _normalized(np.random.default_rng(9).standard_normal((n, 512)).astype(np.float32))
    got, unc = _device_graph(wn, k, 48)
    for j in np.random.default_rng(1).integers(0, n, 24):
        assert np.array_equal(got[j], O.graph_row(wn, int(j), k)), j
    assert unc < n // 100  # the certificate holds for almost every row
