"""Device active-class selection vs the oracle: bit-exact ActiveSets (P=1 layer), both the
padding (mt19937_64 + Lemire + Fisher-Yates) and the over-full (rank/occurrence) branches,
including the golden fixtures generated from the reference."""
import os

import numpy as np
import pytest

import oracle_lib as O
from gpu_util import make_layer, torch_cuda

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _check(n, k, b, m, seed, graph_seed, label_seed, trials=1):
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    g = O.random_graph(n, k, graph_seed)
    shards = [O.compress(g, 1, 0)]
    w = np.ones((n, 128), np.float32)
    layer = make_layer(n, 128, 1, 0, m, b, w, g, precision=X.PREC_FP32_EXACT, seed=seed)
    rng = np.random.default_rng(label_seed)
    for _ in range(trials):
        lab = rng.integers(0, n, b).astype(np.uint32)
        rc, want, ca = O.select_shards("oracle", n, shards, lab, m, seed)
        assert rc == 0
        got, gca = layer.select_active_classes(torch.from_numpy(lab.view(np.int32)).cuda())
        got = got.cpu().numpy().view(np.uint32)
        assert got.size == want.size, (got.size, want.size)
        assert np.array_equal(got, want)
        assert gca == ca
    layer.close()


@pytest.mark.parametrize("m", [10_000, 2_560, 1_000, 300])
def test_select_c1_geometry(m):
    # C1: N=100K, B=256, k=10; M=10% N pads, smaller M exercises the over-full ranking
    _check(100_000, 10, 256, m, 42, 1, m, trials=8)


@pytest.mark.parametrize("seed", [0, 1, 7, 2**63 + 5])
def test_select_seeds(seed):
    _check(20_000, 12, 128, 2_000, seed, 2, 3, trials=4)


def test_select_full_complement():
    # M == N: every class is active (the padding exhausts the complement)
    _check(3_000, 5, 64, 3_000, 9, 4, 5, trials=2)


def test_select_exact_fit():
    # M == |pool| exactly: no padding, no ranking
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    n, k, b = 5_000, 8, 64
    g = O.random_graph(n, k, 6)
    lab = np.random.default_rng(8).integers(0, n, b).astype(np.uint32)
    pool = np.unique(g[lab].ravel())
    m = pool.size
    layer = make_layer(n, 128, 1, 0, m, b, np.ones((n, 128), np.float32), g,
                       precision=X.PREC_FP32_EXACT)
    got, _ = layer.select_active_classes(torch.from_numpy(lab.view(np.int32)).cuda())
    assert np.array_equal(got.cpu().numpy().view(np.uint32), pool.astype(np.uint32))


def test_select_errors():
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    n, k, b = 1_000, 4, 32
    g = O.random_graph(n, k, 1)
    layer = make_layer(n, 128, 1, 0, 8, b, np.ones((n, 128), np.float32), g, precision=X.PREC_FP32_EXACT)
    lab = np.arange(b, dtype=np.uint32)
    with pytest.raises(X.MTooSmall):  # knn_softmax.cpp:24-27
        layer.select_active_classes(torch.from_numpy(lab.view(np.int32)).cuda())
    bad = lab.copy()
    bad[3] = n + 5
    with pytest.raises(X.LabelOutOfRange):
        layer.select_active_classes(torch.from_numpy(bad.view(np.int32)).cuda())


@pytest.mark.parametrize("i", range(9))
def test_select_golden_p1(i):
    z = np.load(os.path.join(GOLDEN, f"select_{i}.npz"))
    if int(z["p"]) != 1:
        pytest.skip("multi-shard fixture: covered by the multi-GPU test")
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    n, k, m = int(z["n"]), int(z["k"]), int(z["m"])
    g = O.random_graph(n, k, int(z["graph_seed"]))
    layer = make_layer(n, 128, 1, 0, m, int(z["b"]), np.ones((n, 128), np.float32), g,
                       precision=X.PREC_FP32_EXACT, seed=int(z["seed"]))
    got, ca = layer.select_active_classes(torch.from_numpy(z["labels"].view(np.int32)).cuda())
    assert np.array_equal(got.cpu().numpy().view(np.uint32), z["active"])


@pytest.mark.parametrize("m", [600, 60])
def test_select_not_self_first(m):
    """Graphs whose lists omit the class itself: labels join the ActiveSet only in the over-full
    branch (knn_softmax.cpp:52-54); contains_all_labels reports the difference."""
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    n, k, b = 2_000, 5, 40
    rng = np.random.default_rng(3)
    g = O.random_graph(n, k + 1, 9)[:, 1:].copy()  # drop self
    shards = [O.compress(g, 1, 0)]
    layer = make_layer(n, 128, 1, 0, m, b, np.ones((n, 128), np.float32), g,
                       precision=X.PREC_FP32_EXACT, seed=5)
    for _ in range(4):
        lab = rng.integers(0, n, b).astype(np.uint32)
        rc, want, ca = O.select_shards("oracle", n, shards, lab, m, 5)
        assert rc == 0
        got, gca = layer.select_active_classes(torch.from_numpy(lab.view(np.int32)).cuda())
        assert np.array_equal(got.cpu().numpy().view(np.uint32), want)
        assert gca == ca
