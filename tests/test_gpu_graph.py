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


def test_graph_many_uncertified_rows():
    """Groups of 20 rows within 1e-4 of each other (half of them exact copies): a row's k-1
    best lie inside its group, closer together than the fp16 certificate can separate, so most
    rows are uncertified and come from the batched exact top-k (many 16-row batches, exact ties
    spanning the 4096-column select chunks, resolved to the lower ids): bit-exact vs the
    oracle."""
    rng = np.random.default_rng(13)
    base = np.repeat(rng.standard_normal((500, 512)).astype(np.float32), 20, axis=0)
    noise = 1e-4 * rng.standard_normal(base.shape).astype(np.float32)
    noise[::2] = 0.0  # exact copies: ties
    w = (base + noise)[rng.permutation(10000)]
    w = np.concatenate([w, rng.standard_normal((2000, 512)).astype(np.float32)])
    wn = _normalized(w)
    got, unc = _device_graph(wn, 12)
    rc, want = O.bruteforce_graph("oracle", wn, 12)
    assert rc == 0 and np.array_equal(got, want)
    assert unc > 32, unc  # the batched exact path ran for several 16-row batches


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


def _dup_weights(seed, n_base, n_rand, scale=0.05):
    """Random rows plus exact and near duplicates (exact score ties, certificate failures)."""
    rng = np.random.default_rng(seed)
    base = rng.standard_normal((n_base, 512)).astype(np.float32)
    w = np.concatenate([base, base, base + 1e-4 * rng.standard_normal((n_base, 512)).astype(np.float32),
                        rng.standard_normal((n_rand, 512)).astype(np.float32)])
    return (w * scale).astype(np.float32)


def test_graph_pilot_chunked_sampled_rows():
    """n > 131072 on one GPU: the pilot seeds the cuts (1-in-32 sample) and the candidate pass
    runs chunk-major over five 32K-column chunks; sampled rows bit-exact vs the oracle."""
    import paper_2102_06025_b200 as X

    n, k = 140_000, 24
    wn = _normalized(np.random.default_rng(21).standard_normal((n, 512)).astype(np.float32))
    got, unc = _device_graph(wn, k, 64)
    for j in np.random.default_rng(4).integers(0, n, 16):
        assert np.array_equal(got[j], O.graph_row(wn, int(j), k)), j
    assert unc < n // 1000
    X.release_graph_cache()  # the cached build scratch goes back to the driver


def test_layer_rebuild_graph_single_gpu():
    """xknn_layer_rebuild_graph == compress_graph(build_graph_bruteforce(l2_normalize_rows(W)))
    and the rebuilt graph drives selection exactly like the reference's."""
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    n, k, m, b = 3000, 12, 300, 64
    w = _dup_weights(11, 200, n - 600)
    wn = _normalized(w)
    rc, g = O.bruteforce_graph("oracle", wn, k)
    assert rc == 0
    kpc, off, flat = O.compress(g, 1, 0)
    layer = X.KnnSoftmaxLayer(n, 512, m_active=m, max_batch=b, rng_seed=42)
    layer.set_weights(torch.from_numpy(w).cuda())
    layer.rebuild_graph(k)
    gk, go, gf = layer.graph()
    assert np.array_equal(gk, kpc) and np.array_equal(go, off) and np.array_equal(gf, flat)
    lab = np.random.default_rng(3).integers(0, n, b).astype(np.uint32)
    act, _ = layer.select_active_classes(torch.from_numpy(lab.view(np.int32)).cuda())
    rc, want, _ = O.select_shards("oracle", n, [(kpc, off, flat)], lab, m, 42)
    assert rc == 0 and np.array_equal(act.cpu().numpy().view(np.uint32), want)
    layer.close()


def test_graph_errors():
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    wn = torch.from_numpy(_normalized(np.random.default_rng(0).standard_normal((300, 512))
                                      .astype(np.float32))).cuda()
    with pytest.raises(X.KTooLarge):
        X.graph_bruteforce(wn, 301)
    with pytest.raises(X.InvalidArgument):
        X.graph_bruteforce(wn, 0)
    with pytest.raises(X.InvalidArgument):  # k' < k (build_graph_ring)
        X.graph_ring(wn, 300, 10, 5, 0, 1)
    g, _ = X.graph_bruteforce(wn, 1)
    assert np.array_equal(g.cpu().numpy()[:, 0], np.arange(300))
    rows, unc, steps = X.graph_ring(wn, 300, 7, 7, 0, 1)
    rc, want = O.bruteforce_graph("oracle", wn.cpu().numpy(), 7)
    assert rc == 0 and np.array_equal(rows.cpu().numpy().view(np.uint32), want) and steps == 0


def test_layer_rebuild_zero_norm_row():
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    w = (np.random.default_rng(1).standard_normal((500, 512)) * 0.05).astype(np.float32)
    w[123] = 0.0
    layer = X.KnnSoftmaxLayer(500, 512, m_active=50, max_batch=16, rng_seed=42)
    layer.set_weights(torch.from_numpy(w).cuda())
    with pytest.raises(X.ZeroNormRow) as ei:
        layer.rebuild_graph(5)
    assert ei.value.row == 123
    layer.close()


def test_rebuild_save_load_roundtrip(tmp_path):
    """rebuild -> rows -> XKNN file -> load_graph on a fresh layer: the same CompressedKnnGraph,
    and the file equals the reference's save_graph of the oracle graph."""
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    n, k = 2000, 9
    w = _dup_weights(3, 100, n - 300)
    layer = X.KnnSoftmaxLayer(n, 512, m_active=200, max_batch=32, rng_seed=42)
    layer.set_weights(torch.from_numpy(w).cuda())
    rows = torch.empty(n, k, dtype=torch.int32, device="cuda")
    layer.rebuild_graph(k, rows_out=rows)
    path = str(tmp_path / "g.xknn")
    X.save_graph_rows(path, n, 0, rows, create=True)
    rc, g = O.bruteforce_graph("oracle", _normalized(w), k)
    assert rc == 0 and np.array_equal(rows.cpu().numpy().view(np.uint32), g)
    fresh = X.KnnSoftmaxLayer(n, 512, m_active=200, max_batch=32, rng_seed=42)
    assert fresh.load_graph(path) == k
    for a, b in zip(fresh.graph(), layer.graph()):
        assert np.array_equal(a, b)
    layer.close()
    fresh.close()


@pytest.mark.parametrize("d", [512, 128])
def test_classify_retrieval(d):
    """classify_retrieval == argmax of the reference-order cosine (oracle restatement of
    SPEC.md:568-576), ties to the lower id; a query equal to w_j returns j."""
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    n = 5000 if d == 512 else 700
    rng = np.random.default_rng(d)
    w = (rng.standard_normal((n, d)) * 0.05).astype(np.float32)
    w[n - 1] = w[17]  # exact duplicate class: ties resolve to the lower id
    q = np.concatenate([rng.standard_normal((300, d)).astype(np.float32), w[[3, 17, n - 1, 4000 % n]] * 3.0])
    layer = X.KnnSoftmaxLayer(n, d, m_active=n // 10, max_batch=16, rng_seed=42,
                              precision=X.PREC_BF16 if d == 512 else X.PREC_FP32_EXACT)
    layer.set_weights(torch.from_numpy(w).cuda())
    cls, sc = layer.classify(torch.from_numpy(q).cuda())
    rc, want, wsc = O.classify_retrieval(q, w)
    assert rc == 0
    assert np.array_equal(cls.cpu().numpy().view(np.uint32), want)
    assert np.array_equal(sc.cpu().numpy(), wsc)
    assert list(want[-4:]) == [3, 17, 17, 4000 % n]
    layer.close()
