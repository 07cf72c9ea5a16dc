"""The reference's single-device free functions of the path on device, against the oracle:
select_active_classes over the full KnnGraph (knn_softmax.cpp:100-115; ranks = positions in the
full lists, not the shard slices), the span<CompressedKnnGraph> overload with P shards on one
device (merged slices with per-entry ranks), and knn_softmax_forward_backward
(knn_softmax.cpp:136-186, fp32 in the reference's summation order)."""
import numpy as np
import pytest

import oracle_lib as O
from gpu_util import rel_err, torch_cuda

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,k,b,m", [(20_000, 12, 128, 2_000), (5_000, 8, 300, 500),
                                     (3_000, 6, 64, 3_000)])
def test_select_full_graph(n, k, b, m):
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    g = O.random_graph(n, k, 3)
    gd = torch.from_numpy(g.view(np.int32)).cuda()
    rng = np.random.default_rng(n)
    for _ in range(3):
        lab = rng.integers(0, n, b).astype(np.uint32)
        got, ca = X.select_active_classes_full(gd, torch.from_numpy(lab.view(np.int32)).cuda(), m, 42)
        rc, want, ca_or = O.select_full("oracle", g, lab, m, 42)
        assert rc == 0
        assert np.array_equal(got.cpu().numpy().view(np.uint32), want)
        assert ca == ca_or
    with pytest.raises(X.LabelOutOfRange):
        bad = lab.copy()
        bad[0] = n
        X.select_active_classes_full(gd, torch.from_numpy(bad.view(np.int32)).cuda(), m, 42)
    with pytest.raises(X.MTooSmall):
        X.select_active_classes_full(gd, torch.from_numpy(lab.view(np.int32)).cuda(), 3, 42)


@pytest.mark.parametrize("p,m", [(3, 400), (4, 4_000), (2, 150)])
def test_select_span_of_shards_one_device(p, m):
    """select_active_classes(span<CompressedKnnGraph>) with P shards held by one layer: each
    label's P slices concatenated, ranks within their own slice -- both branches."""
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    n, k, b = 12_000, 10, 96
    g = O.random_graph(n, k, 8)
    shards = [O.compress(g, p, s) for s in range(p)]
    kpc = np.zeros(n, np.uint32)
    flat, rank = [], []
    for c in range(n):
        for (kp, off, fl) in shards:
            sl = fl[int(off[c]):int(off[c]) + int(kp[c])]
            flat.append(sl)
            rank.append(np.arange(sl.size, dtype=np.uint32))
            kpc[c] += sl.size
    flat = np.concatenate(flat).astype(np.uint32)
    rank = np.concatenate(rank).astype(np.uint32)
    off = np.zeros(n, np.uint64)
    off[1:] = np.cumsum(kpc[:-1].astype(np.uint64))
    layer = X.KnnSoftmaxLayer(n, 128, m_active=m, max_batch=b, rng_seed=5,
                              precision=X.PREC_FP32_EXACT, select_only=True)
    layer.set_shard_graph_ranked(*(torch.from_numpy(a.view(t)).cuda() for a, t in
                                   ((kpc, np.int32), (off, np.int64), (flat, np.int32),
                                    (rank, np.int32))))
    rng = np.random.default_rng(p)
    for _ in range(4):
        lab = rng.integers(0, n, b).astype(np.uint32)
        got, ca = layer.select_active_classes(torch.from_numpy(lab.view(np.int32)).cuda())
        rc, want, ca_or = O.select_shards("oracle", n, shards, lab, m, 5)
        assert rc == 0
        assert np.array_equal(got.cpu().numpy().view(np.uint32), want)
        assert ca == ca_or
    with pytest.raises(X.Unsupported):
        layer.weights()
    layer.close()


@pytest.mark.parametrize("n,b,m,d", [(20_000, 128, 2_000, 512), (3_000, 33, 3_000, 256),
                                     (5_000, 1, 40, 128)])
def test_knn_softmax_forward_backward(n, b, m, d):
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    rng = np.random.default_rng(n + b)
    _, x, _, _ = O.l2_normalize(rng.standard_normal((b, d)).astype(np.float32))
    _, w, _, _ = O.l2_normalize(rng.standard_normal((n, d)).astype(np.float32))
    act = np.sort(rng.choice(n, m, replace=False)).astype(np.uint32)
    lab = act[rng.integers(0, m, b)]
    rc, loss_or, gl_or, gf_or, gw_or = O.knn_softmax_fwd_bwd("oracle", x, w, lab, act, 30.0)
    assert rc == 0
    t = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    loss, gl, gf, gw = X.knn_softmax_forward_backward(t(x), t(w), t(lab.view(np.int32)),
                                                      t(act.view(np.int32)), 30.0)
    assert abs(loss - loss_or) <= 1e-5 * abs(loss_or)
    assert rel_err(gl.cpu().numpy(), gl_or) <= 1e-5
    assert rel_err(gf.cpu().numpy(), gf_or) <= 1e-5
    assert rel_err(gw.cpu().numpy(), gw_or) <= 1e-5
    bad = lab.copy()
    bad[0] = np.setdiff1d(np.arange(n), act)[0] if m < n else lab[0]
    if m < n:
        with pytest.raises(X.LabelNotActive):
            X.knn_softmax_forward_backward(t(x), t(w), t(bad.view(np.int32)), t(act.view(np.int32)), 30.0)


def test_in_place_graph_install_matches_copy():
    """xknn_layer_graph_buffers + xknn_layer_graph_commit (bench.py's in-place install) installs
    the same CompressedKnnGraph as xknn_layer_set_graph_csr, and selection agrees."""
    import paper_2102_06025_b200 as X
    import bench

    torch = torch_cuda()
    n, k, b, m = 50_000, 8, 128, 5_000
    a = X.KnnSoftmaxLayer(n, 128, m_active=m, max_batch=b, rng_seed=3,
                          precision=X.PREC_FP32_EXACT, select_only=True)
    bench.install_shard_graph(torch, a, n, k, 1, 0, seed=5, chunk=7_000)
    kpc, off, flat = a.graph()
    g = np.zeros((n, k), np.uint32)
    for c in range(n):
        g[c] = flat[int(off[c]):int(off[c]) + int(kpc[c])]
    assert (kpc == k).all() and (g[:, 0] == np.arange(n)).all()
    shards = [O.compress(g, 1, 0)]
    lab = np.random.default_rng(1).integers(0, n, b).astype(np.uint32)
    got, _ = a.select_active_classes(torch.from_numpy(lab.view(np.int32)).cuda())
    rc, want, _ = O.select_shards("oracle", n, shards, lab, m, 3)
    assert rc == 0 and np.array_equal(got.cpu().numpy().view(np.uint32), want)
    a.close()
