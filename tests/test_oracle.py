"""The CPU oracle (oracle/xknn_oracle.c) against the SPEC.md known answers, the committed golden
fixtures (generated from the compiled reference by tests/golden/make_golden.py) and, when
oracle/_ref is built, against the reference itself on fresh seeded inputs."""
import math
import os

import numpy as np
import pytest

import oracle_lib as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- SPEC.md known answers
def test_kat_l2_normalize():
    rc, out, norms, _ = O.l2_normalize(np.array([[3, 4]], np.float32))
    assert rc == 0 and np.allclose(out, [[0.6, 0.8]]) and norms[0] == 5.0
    rc, out, _, _ = O.l2_normalize(np.array([[1, 0, 0]], np.float32))
    assert rc == 0 and np.array_equal(out, [[1, 0, 0]])
    rc, _, _, bad = O.l2_normalize(np.array([[1, 1], [0, 0]], np.float32))
    assert rc == 2 and bad == 1  # ZeroNormRow(1)


def test_kat_softmax_xent():
    rc, loss, grad = O.softmax_xent("oracle", np.zeros((1, 2), np.float32), np.array([0]))
    assert rc == 0 and abs(loss - math.log(2)) < 1e-12
    assert abs(grad.sum()) < 1e-7
    rc, loss, _ = O.softmax_xent("oracle", np.array([[1000, 0]], np.float32), np.array([0]))
    assert rc == 0 and abs(loss) < 1e-12
    rc, _, _ = O.softmax_xent("oracle", np.zeros((1, 2), np.float32), np.array([2]))
    assert rc == 3  # LabelOutOfRange


def test_kat_bruteforce_graph():
    rc, g = O.bruteforce_graph("oracle", np.eye(3, dtype=np.float32), 1)
    assert rc == 0 and g.ravel().tolist() == [0, 1, 2]
    rc, g = O.bruteforce_graph("oracle", np.array([[1, 0], [1, 0]], np.float32), 2)
    assert rc == 0 and g.tolist() == [[0, 1], [1, 0]]
    rc, _ = O.bruteforce_graph("oracle", np.eye(3, dtype=np.float32), 4)
    assert rc == 4  # KTooLarge


def test_kat_compress_offsets():
    g = np.array([[0, 1, 2], [1, 0, 2], [2, 0, 1]], np.uint32)
    kpc, off, flat = O.compress(g, 1, 0)
    assert kpc.tolist() == [3, 3, 3] and off.tolist() == [0, 3, 6] and flat.size == 9
    kpc, off, flat = O.compress(g, 3, 1)  # shard 1 owns class 1 only
    assert kpc.tolist() == [1, 1, 1] and off.tolist() == [0, 1, 2] and flat.tolist() == [1, 1, 1]


def test_kat_selection():
    g = O.random_graph(50, 3, 0)
    lab = np.full(8, 7, np.uint32)
    rc, act, ca = O.select_full("oracle", g, lab, 3, 0)
    assert rc == 0 and act.tolist() == sorted(g[7].tolist()) and ca
    rc, act, _ = O.select_full("oracle", g, lab, 50, 0)  # M == N: full softmax
    assert act.tolist() == list(range(50))
    rc, _, _ = O.select_full("oracle", g, np.arange(5, dtype=np.uint32), 4, 0)
    assert rc == 6  # MTooSmall
    rc, act, _ = O.select_full("oracle", g, np.arange(5, dtype=np.uint32), 20, 9)
    assert rc == 0 and act.size == 20 and len(set(act.tolist())) == 20
    pool = set(g[:5].ravel().tolist())
    assert pool <= set(act.tolist())  # padding is disjoint from and added to the pool


def test_mt19937_64_known_answer():
    # C++11 [rand.predef]: the 10000th output of default-seeded mt19937_64 is 9981545732273789042
    s = O.mt64_stream(5489, 10000)
    assert int(s[-1]) == 9981545732273789042


# ---------------------------------------------------------------- golden fixtures (from _ref)
@pytest.mark.parametrize("i", range(9))
def test_golden_selection(i):
    z = np.load(os.path.join(GOLDEN, f"select_{i}.npz"))
    n, k, p = int(z["n"]), int(z["k"]), int(z["p"])
    g = O.random_graph(n, k, int(z["graph_seed"]))
    shards = [O.compress(g, p, s) for s in range(p)]
    rc, act, ca = O.select_shards("oracle", n, shards, z["labels"], int(z["m"]), int(z["seed"]))
    assert rc == 0
    assert np.array_equal(act, z["active"]) and ca == bool(z["contains_all"])


def test_golden_fc_step():
    z = np.load(os.path.join(GOLDEN, "fc_step.npz"))
    n, d, k, m, p = (int(z[c]) for c in ("n", "d", "k", "m", "p"))
    rng = np.random.default_rng(int(z["w_seed"]))
    w = (rng.standard_normal((n, d)) * 0.05).astype(np.float32)
    g = O.random_graph(n, k, int(z["graph_seed"]))
    shards = [O.compress(g, p, s) for s in range(p)]
    v = np.zeros_like(w)
    for t in range(z["x"].shape[0]):
        rc, loss, *_ = O.fc_train_step(w, v, z["x"][t], z["labels"][t], shards, m, 42)
        assert rc == 0 and loss == z["losses"][t]  # bit-exact
    assert np.array_equal(w, z["w_final"])


def test_golden_bruteforce_graph():
    z = np.load(os.path.join(GOLDEN, "graph_bf.npz"))
    _, wn, _, _ = O.l2_normalize(z["w"])
    rc, g = O.bruteforce_graph("oracle", wn, int(z["k"]))
    assert rc == 0 and np.array_equal(g, z["graph"])


# ---------------------------------------------------------------- live reference (oracle/_ref)
@pytest.mark.ref
@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_ref_selection_random(p):
    rng = np.random.default_rng(100 + p)
    for trial in range(25):
        n = int(rng.integers(50, 6000))
        k = int(rng.integers(1, min(n, 40)))
        b = int(rng.integers(1, 200))
        g = O.random_graph(n, k, trial)
        shards = [O.compress(g, p, s) for s in range(p)]
        lab = rng.integers(0, n, b).astype(np.uint32)
        m = int(rng.integers(1, n + 1))
        seed = int(rng.integers(0, 2**63))
        a = O.select_shards("oracle", n, shards, lab, m, seed)
        r = O.select_shards("ref", n, shards, lab, m, seed)
        assert a[0] == r[0]
        if a[0] == 0:
            assert np.array_equal(a[1], r[1]) and a[2] == r[2]


@pytest.mark.ref
@pytest.mark.parametrize("p", [1, 2, 4])
def test_ref_fc_step_and_feature_grad(p):
    rng = np.random.default_rng(7 + p)
    n, d, b, k, m = 4000, 64, 48, 8, 400
    w = (rng.standard_normal((n, d)) * 0.05).astype(np.float32)
    g = O.random_graph(n, k, p)
    shards = [O.compress(g, p, s) for s in range(p)]
    sim = O.RefSim(w, p)
    sim.set_graphs(shards)
    w2, v2 = w.copy(), np.zeros_like(w)
    for _ in range(3):
        x = rng.standard_normal((b, d)).astype(np.float32)
        lab = rng.integers(0, n, b).astype(np.uint32)
        w_before = w2.copy()
        rc, loss_r, na = sim.step(x, lab, m, 42)
        rc2, loss_o, act, gfeat, _ = O.fc_train_step(w2, v2, x, lab, shards, m, 42)
        assert rc == 0 and rc2 == 0 and na == act.size
        assert loss_r == loss_o
        assert np.array_equal(sim.weights(), w2)
        rc3, loss3, gref = O.ref_feature_grad(w_before, x, lab, act, p)
        assert rc3 == 0 and loss3 == loss_o and np.array_equal(gref, gfeat)


def _micro_rows(b, p, micro):
    """Rank-major row lists of each micro-batch (parallel.cpp:514-523)."""
    sl = b // p
    mc = min(micro, sl)
    base, rem = divmod(sl, mc)
    out, off = [], 0
    for c in range(mc):
        rc = base + (1 if c < rem else 0)
        out.append(np.array([w * sl + off + i for w in range(p) for i in range(rc)]))
        off += rc
    return out


def test_oracle_micro_step_one_micro_is_the_plain_step():
    rng = np.random.default_rng(3)
    n, d, b, k, m, p = 3000, 64, 40, 6, 300, 2
    w = (rng.standard_normal((n, d)) * 0.05).astype(np.float32)
    g = O.random_graph(n, k, 9)
    shards = [O.compress(g, p, s) for s in range(p)]
    x = rng.standard_normal((b, d)).astype(np.float32)
    lab = rng.integers(0, n, b).astype(np.uint32)
    w1, v1, w2, v2 = w.copy(), np.zeros_like(w), w.copy(), np.zeros_like(w)
    rc1, l1, a1, g1, _ = O.fc_train_step(w1, v1, x, lab, shards, m, 5)
    rc2, l2, a2, g2 = O.fc_train_step_mb(w2, v2, x, lab, shards, m, 5, 1)
    assert rc1 == rc2 == 0 and l1 == l2 and np.array_equal(a1, a2)
    assert np.array_equal(w1, w2) and np.array_equal(v1, v2) and np.array_equal(g1, g2)


@pytest.mark.ref
@pytest.mark.parametrize("p,micro", [(1, 2), (1, 5), (2, 3), (4, 2)])
def test_ref_fc_step_micro_batches(p, micro):
    """StepOptions::micro_batches > 1 (parallel.cpp:444, :505-591): the oracle matches the stock
    HybridSim bit for bit in loss and weights, and its per-micro-batch feature gradient matches
    the reference's free functions composed on each micro-batch."""
    rng = np.random.default_rng(17 + p + micro)
    n, d, b, k, m = 4000, 64, 48, 8, 400
    w = (rng.standard_normal((n, d)) * 0.05).astype(np.float32)
    g = O.random_graph(n, k, p)
    shards = [O.compress(g, p, s) for s in range(p)]
    sim = O.RefSim(w, p)
    sim.set_graphs(shards)
    w2, v2 = w.copy(), np.zeros_like(w)
    for _ in range(2):
        x = rng.standard_normal((b, d)).astype(np.float32)
        lab = rng.integers(0, n, b).astype(np.uint32)
        w_before = w2.copy()
        rc, loss_r, na = sim.step_mb(x, lab, m, 42, micro)
        rc2, loss_o, act, gfeat = O.fc_train_step_mb(w2, v2, x, lab, shards, m, 42, micro)
        assert rc == 0 and rc2 == 0 and na == act.size
        assert loss_r == loss_o
        assert np.array_equal(sim.weights(), w2)
        for rows in _micro_rows(b, p, micro):
            rc3, _, gref = O.ref_feature_grad(w_before, x[rows], lab[rows], act, p)
            assert rc3 == 0 and np.array_equal(gref, gfeat[rows])


@pytest.mark.ref
def test_ref_graph_builders():
    rng = np.random.default_rng(1)
    w = rng.standard_normal((400, 24)).astype(np.float32)
    _, wn, _, _ = O.l2_normalize(w)
    rc, go = O.bruteforce_graph("oracle", wn, 10)
    rc2, gr = O.bruteforce_graph("ref", wn, 10)
    assert rc == rc2 == 0 and np.array_equal(go, gr)


@pytest.mark.ref
def test_ref_selection_not_self_first():
    rng = np.random.default_rng(11)
    for trial in range(20):
        n = int(rng.integers(100, 3000))
        k = int(rng.integers(2, 12))
        g = O.random_graph(n, k + 1, trial)[:, 1:].copy()
        p = int(rng.choice([1, 2, 4]))
        shards = [O.compress(g, p, s) for s in range(p)]
        lab = rng.integers(0, n, 30).astype(np.uint32)
        m = int(rng.integers(30, n))
        a = O.select_shards("oracle", n, shards, lab, m, trial)
        r = O.select_shards("ref", n, shards, lab, m, trial)
        assert a[0] == r[0] and np.array_equal(a[1], r[1]) and a[2] == r[2]


def _py_select_pad_stream(n, pool, m, words):
    """Pure-Python finish_selection padding branch (knn_softmax.cpp:33-51) over an injected word
    stream with libstdc++'s Lemire draw (uniform_int_dist.h:257-274) -- small cases only."""
    comp = [c for c in range(n) if c not in pool]
    sel = sorted(pool)
    it = iter(int(w) for w in words)
    for i in range(m - len(pool)):
        rng_ = len(comp) - i
        prod = next(it, 0) * rng_
        low = prod & (2**64 - 1)
        if low < rng_:
            thr = (2**64 - rng_) % rng_
            while low < thr:
                prod = next(it, 0) * rng_
                low = prod & (2**64 - 1)
        j = i + (prod >> 64)
        comp[i], comp[j] = comp[j], comp[i]
        sel.append(comp[i])
    return np.array(sorted(sel), np.uint32)


def test_oracle_injected_stream():
    """or_select_active_shards_stream: the true mt19937_64 words reproduce the seeded selection,
    and zero words take the Lemire rejection loop exactly as a Python restatement does."""
    n, k, b, m = 3_000, 6, 40, 600
    g = O.random_graph(n, k, 2)
    shards = [O.compress(g, 1, 0)]
    lab = np.random.default_rng(1).integers(0, n, b).astype(np.uint32)
    words = O.mt64_stream(5, m + 64)
    rc, a, _ = O.select_shards("oracle", n, shards, lab, m, 5)
    rc2, b_, _ = O.select_shards_stream(n, shards, lab, m, words)
    assert rc == rc2 == 0 and np.array_equal(a, b_)
    pool = set(int(c) for c in np.unique(g[lab].ravel()))
    words[[2, 7, 8]] = 0
    rc, c_, _ = O.select_shards_stream(n, shards, lab, m, words)
    assert rc == 0 and not np.array_equal(a, c_)
    assert np.array_equal(c_, _py_select_pad_stream(n, pool, m, words))


def test_graph_row_checker_streamed():
    """GraphRowChecker (chunks streamed in any order) == graph_row on the whole matrix."""
    rng = np.random.default_rng(4)
    n, d, k = 3_000, 64, 12
    rc, wn, _, _ = O.l2_normalize(rng.standard_normal((n, d)).astype(np.float32))
    wn[17] = wn[900]  # an exact duplicate: a score tie resolved by index
    qid = np.array([0, 17, 900, 2999, 1234])
    chk = O.GraphRowChecker(qid, wn[qid], k)
    for c0 in (2000, 0, 1000):  # out of order
        chk.update(wn[c0:c0 + 1000], c0)
    got = chk.rows()
    for a, j in enumerate(qid):
        assert np.array_equal(got[a], O.graph_row(wn, int(j), k))


@pytest.mark.ref
def test_oracle_knn_softmax_fwd_bwd_vs_reference():
    """or_knn_softmax_forward_backward is bit-identical with the compiled reference's
    knn_softmax_forward_backward (knn_softmax.cpp:136-186), including its errors."""
    rng = np.random.default_rng(6)
    n, d, b, m = 700, 128, 33, 90
    _, x, _, _ = O.l2_normalize(rng.standard_normal((b, d)).astype(np.float32))
    _, w, _, _ = O.l2_normalize(rng.standard_normal((n, d)).astype(np.float32))
    act = np.sort(rng.choice(n, m, replace=False)).astype(np.uint32)
    lab = act[rng.integers(0, m, b)]
    a = O.knn_softmax_fwd_bwd("oracle", x, w, lab, act)
    r = O.knn_softmax_fwd_bwd("ref", x, w, lab, act)
    assert a[0] == r[0] == 0 and a[1] == r[1]
    for i in (2, 3, 4):
        assert np.array_equal(a[i], r[i])
    bad = lab.copy()
    bad[5] = np.setdiff1d(np.arange(n), act)[0]
    assert O.knn_softmax_fwd_bwd("oracle", x, w, bad, act)[0] == 7  # LabelNotActive
    assert O.knn_softmax_fwd_bwd("ref", x, w, bad, act)[0] == 7
