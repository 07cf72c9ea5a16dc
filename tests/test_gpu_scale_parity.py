"""Parity at the benchmarked geometries (BASELINE configs[1..3]) and on the rare draw path.

* Selection at C2 (N=1M, B=1024, k=50, M=100K), C3 at P=1 (N=10M, B=4096, k=100, M=1M) and the
  C4 per-rank proxy (N=12.5M, B=8192, k=100, M=1.25M): bit-exact ActiveSets vs the oracle
  (select_active_classes(span<CompressedKnnGraph>), knn_softmax.cpp:117-134 + :17-81).  The
  graphs are generated on the device; the oracle gets the labels' rows (the only ones selection
  reads).
* The Lemire rejection loop of uniform_int_distribution (uniform_int_dist.h:268-272), which a
  real mt19937_64 stream hits with probability ~ need*csize/2^64: driven with crafted word
  streams (zero words are always rejected) through xknn_layer_set_draw_stream, against the
  oracle fed the same words.
* One fc train step at C2 in both precisions vs the oracle (bit-exact with the reference's
  HybridSim, tests/test_oracle.py); measured errors are recorded (parity_record).
"""
import numpy as np
import pytest

import oracle_lib as O
from gpu_util import (BF16_GRAD, BF16_LOSS, device_graph, host_label_csr, make_layer,
                      parity_record, rel_err, torch_cuda)

pytestmark = pytest.mark.gpu


def _select_geometry(n, b, k, m, trials, seed=42):
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    flat, kpc, off = device_graph(n, k, 11)
    layer = X.KnnSoftmaxLayer(n, 512, m_active=m, max_batch=b, rng_seed=seed,
                              precision=X.PREC_BF16)
    layer.set_shard_graph(kpc, off, flat)
    rng = np.random.default_rng(n + b)
    for t in range(trials):
        lab = rng.integers(0, n, b).astype(np.uint32)
        got, ca = layer.select_active_classes(torch.from_numpy(lab.view(np.int32)).cuda())
        got = got.cpu().numpy().view(np.uint32)
        rc, want, ca_or = O.select_shards("oracle", n, [host_label_csr(flat, n, k, lab)], lab, m,
                                          seed)
        assert rc == 0
        assert got.size == want.size == m
        assert np.array_equal(got, want), f"trial {t}: first diff at {np.argmax(got != want)}"
        assert ca == ca_or
    layer.close()
    del flat, kpc, off
    torch.cuda.empty_cache()


def test_select_c2_geometry():
    _select_geometry(1_000_000, 1024, 50, 100_000, trials=3)


def test_select_c3_geometry_p1():
    _select_geometry(10_000_000, 4096, 100, 1_000_000, trials=2)


def test_select_c4_per_rank_proxy():
    # one rank of C4 (100M classes over 8 GPUs): 12.5M classes, B = 8192, k = 100, M_w = 1.25M
    _select_geometry(12_500_000, 8192, 100, 1_250_000, trials=1)


@pytest.mark.parametrize("zeros", [[0], [3, 4, 5], [17, 1000, 1001, 4095]])
def test_select_lemire_rejection_replay(zeros):
    """k_picks flags the first rejected draw and k_picks_replay redraws sequentially from it."""
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    n, k, b, m = 50_000, 10, 256, 5_000
    g = O.random_graph(n, k, 5)
    shards = [O.compress(g, 1, 0)]
    layer = make_layer(n, 128, 1, 0, m, b, np.ones((n, 128), np.float32), g,
                       precision=X.PREC_FP32_EXACT, seed=9)
    words = O.mt64_stream(9, m + 64)
    words[zeros] = 0
    layer.set_draw_stream(words)
    rng = np.random.default_rng(3)
    for _ in range(3):
        lab = rng.integers(0, n, b).astype(np.uint32)
        got, ca = layer.select_active_classes(torch.from_numpy(lab.view(np.int32)).cuda())
        got = got.cpu().numpy().view(np.uint32)
        rc, want, ca_or = O.select_shards_stream(n, shards, lab, m, words)
        assert rc == 0
        assert np.array_equal(got, want)
        # the injected zeros changed the draw (the replay path really ran)
        rc, plain, _ = O.select_shards("oracle", n, shards, lab, m, 9)
        assert not np.array_equal(plain, want)
    layer.set_draw_stream(None)  # back to mt19937_64(rng_seed)
    lab = rng.integers(0, n, b).astype(np.uint32)
    got, _ = layer.select_active_classes(torch.from_numpy(lab.view(np.int32)).cuda())
    rc, want, _ = O.select_shards("oracle", n, shards, lab, m, 9)
    assert np.array_equal(got.cpu().numpy().view(np.uint32), want)
    layer.close()


def _c2_step(precision, steps):
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    n, d, b, k, m = 1_000_000, 512, 1024, 50, 100_000
    rng = np.random.default_rng(2)
    w = (rng.standard_normal((n, d), dtype=np.float32) * np.float32(0.05)).astype(np.float32)
    g = O.random_graph(n, k, 4)
    shards = [O.compress(g, 1, 0)]
    layer = make_layer(n, d, 1, 0, m, b, w, g, precision=precision, seed=42)
    w_or, v_or = w.copy(), np.zeros_like(w)
    errs = []
    for _ in range(steps):
        x = rng.standard_normal((b, d), dtype=np.float32)
        lab = rng.integers(0, n, b).astype(np.uint32)
        rc, loss_or, act, gf_or, _ = O.fc_train_step(w_or, v_or, x, lab, shards, m, 42)
        assert rc == 0 and act.size == m
        gf = torch.empty(b, d, device="cuda")
        loss = layer.train_step(torch.from_numpy(x).cuda(),
                                torch.from_numpy(lab.view(np.int32)).cuda(), 0.1,
                                grad_features_local=gf)
        gfn = gf.cpu().numpy()
        errs.append(dict(loss_rel=abs(loss - loss_or) / abs(loss_or),
                         gf_relF=rel_err(gfn, gf_or),
                         gf_maxovermax=float(np.abs(gfn - gf_or).max() / np.abs(gf_or).max())))
    wg = layer.weights().cpu().numpy()
    vg = layer.velocity().cpu().numpy()
    layer.close()
    upd, upd_or = wg - w, w_or - w
    res = dict(steps=errs, update_relF=rel_err(upd, upd_or),
               update_maxovermax=float(np.abs(upd - upd_or).max() / np.abs(upd_or).max()),
               velocity_relF=rel_err(vg, v_or))
    untouched = np.all(w_or == w, axis=1)
    assert np.array_equal(wg[untouched], w[untouched])
    return res


def test_step_c2_bf16():
    import paper_2102_06025_b200 as X

    r = _c2_step(X.PREC_BF16, 2)
    parity_record("c2_bf16", **r)
    for e in r["steps"]:
        assert e["loss_rel"] <= BF16_LOSS
        assert e["gf_relF"] <= BF16_GRAD
    assert r["update_relF"] <= BF16_GRAD


def test_step_c2_fp32_exact():
    import paper_2102_06025_b200 as X

    r = _c2_step(X.PREC_FP32_EXACT, 1)
    parity_record("c2_fp32_exact", **r)
    for e in r["steps"]:
        assert e["loss_rel"] <= 1e-5
        assert e["gf_relF"] <= 1e-5
    assert r["update_relF"] <= 1e-5
    assert r["velocity_relF"] <= 1e-5


def test_step_c2_fp32_tensor_cores():
    import paper_2102_06025_b200 as X

    r = _c2_step(X.PREC_FP32, 2)
    parity_record("c2_fp32tc", **r)
    for e in r["steps"]:
        assert e["loss_rel"] <= 1e-5
        assert e["gf_relF"] <= 1e-5
    assert r["update_relF"] <= 1e-5
    assert r["velocity_relF"] <= 1e-5
