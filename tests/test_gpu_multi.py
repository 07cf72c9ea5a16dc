"""Class-sharded layer over NCCL on P GPUs vs the oracle at the same shard count P.

Selection is bit-exact per shard (the rank-order concatenation is the reference ActiveSet);
loss, weights and feature gradients within the precision's bound (test_gpu_step.py)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle_lib as O
from gpu_util import BF16_GRAD, BF16_LOSS, parity_record, rel_err

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _ngpus():
    import torch

    return torch.cuda.device_count()


@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("m", [4_000, 400])  # padding branch / over-full ranking branch
@pytest.mark.parametrize("precision,tol_loss,tol_g", [("fp32", 1e-5, 1e-5), ("fp32tc", 1e-5, 1e-5),
                                                     ("bf16", BF16_LOSS, BF16_GRAD)])
def test_multi_gpu_step(p, m, precision, tol_loss, tol_g, tmp_path):
    if _ngpus() < p:
        pytest.skip(f"needs {p} GPUs")
    n, b, k, steps = 40_003, 256, 10, 2  # shards of unequal size (ShardLayout remainder)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={p}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + p + (m % 97)}",
           os.path.join(HERE, "mp_worker.py"), "--out", str(tmp_path), "--num-classes", str(n), "--batch",
           str(b), "--knn", str(k), "--m-active", str(m), "--steps", str(steps), "--precision", precision]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [np.load(os.path.join(tmp_path, f"rank{i}.npz")) for i in range(p)]

    from mp_worker import problem

    w, g = problem(n, 512, k, 7)
    shards = [O.compress(g, p, s) for s in range(p)]
    w_or, v_or = w.copy(), np.zeros_like(w)
    rng = np.random.default_rng(99)
    for s in range(steps):
        x = rng.standard_normal((b, 512)).astype(np.float32)
        lab = rng.integers(0, n, b).astype(np.uint32)
        rc, want, ca = O.select_shards("oracle", n, shards, lab, m, 42)
        assert rc == 0
        got = np.concatenate([r[f"active_{s}"] for r in res])
        assert np.array_equal(got, want)  # bit-exact ActiveSet across shards
        assert all(bool(r[f"contains_{s}"]) for r in res) == ca
        rc, loss_or, act, gf_or, _ = O.fc_train_step(w_or, v_or, x, lab, shards, m, 42)
        assert rc == 0 and np.array_equal(act, want)
        for r in res:
            assert abs(float(r[f"loss_{s}"]) - loss_or) <= tol_loss * abs(loss_or)
        gf = np.concatenate([r[f"gf_{s}"] for r in res])
        assert rel_err(gf, gf_or) <= tol_g
    wg = np.concatenate([r["w"] for r in res])
    assert rel_err(wg - w, w_or - w) <= tol_g
    untouched = np.all(w_or == w, axis=1)
    assert np.array_equal(wg[untouched], w[untouched])


@pytest.mark.parametrize("p", [2, 4])
@pytest.mark.parametrize("precision,tol_loss,tol_g", [("fp32tc", 1e-5, 1e-5),
                                                     ("bf16", BF16_LOSS, BF16_GRAD)])
def test_multi_gpu_step_c2(p, precision, tol_loss, tol_g, tmp_path):
    """One step at the benchmarked C2 geometry (N = 1M, B = 1024, k = 50, M = 100K -- bench.py's
    workload at every N) class-sharded over P GPUs vs the oracle at the same P: bit-exact
    ActiveSet, loss / feature gradient / weight update within the precision's bound, the same
    set of updated rows."""
    if _ngpus() < p:
        pytest.skip(f"needs {p} GPUs")
    n, b, k, m = 1_000_000, 1024, 50, 100_000
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={p}",
           "--master-addr=127.0.0.1", f"--master-port={29620 + p}",
           os.path.join(HERE, "mp_worker.py"), "--out", str(tmp_path), "--num-classes", str(n),
           "--batch", str(b), "--knn", str(k), "--m-active", str(m), "--steps", "1",
           "--precision", precision, "--compact"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [np.load(os.path.join(tmp_path, f"rank{i}.npz")) for i in range(p)]

    from mp_worker import problem

    w, g = problem(n, 512, k, 7)
    shards = [O.compress(g, p, s) for s in range(p)]
    w_or, v_or = w.copy(), np.zeros_like(w)
    rng = np.random.default_rng(99)
    x = rng.standard_normal((b, 512)).astype(np.float32)
    lab = rng.integers(0, n, b).astype(np.uint32)
    rc, loss_or, act, gf_or, _ = O.fc_train_step(w_or, v_or, x, lab, shards, m, 42)
    assert rc == 0
    assert np.array_equal(np.concatenate([r["active_0"] for r in res]), act)
    for r in res:
        assert abs(float(r["loss_0"]) - loss_or) <= tol_loss * abs(loss_or)
    assert rel_err(np.concatenate([r["gf_0"] for r in res]), gf_or) <= tol_g
    rows = np.concatenate([r["w_rows"] + int(r["begin"]) for r in res])
    assert np.array_equal(rows, np.flatnonzero(np.any(w_or != w, axis=1)))  # same rows touched
    delta = np.concatenate([r["w_delta"] for r in res])
    e = rel_err(delta, (w_or - w)[rows])
    parity_record(f"multi_c2_{precision}_p{p}", loss_rel=abs(float(res[0]["loss_0"]) - loss_or) / abs(loss_or),
                  update_relF=e)
    assert e <= tol_g


@pytest.mark.parametrize("p,micro", [(2, 3), (4, 2)])
def test_multi_gpu_micro_batches(p, micro, tmp_path):
    """StepOptions::micro_batches over P ranks: each rank's slice splits into the same balanced
    micro-batches (parallel.cpp:514-523); loss, weights and the micro-scaled feature gradients
    against the oracle's micro-batch step."""
    if _ngpus() < p:
        pytest.skip(f"needs {p} GPUs")
    n, b, k, m, steps = 40_003, 240, 10, 4_000, 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={p}",
           "--master-addr=127.0.0.1", f"--master-port={29580 + p}",
           os.path.join(HERE, "mp_worker.py"), "--out", str(tmp_path), "--num-classes", str(n),
           "--batch", str(b), "--knn", str(k), "--m-active", str(m), "--steps", str(steps),
           "--precision", "bf16", "--micro", str(micro)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [np.load(os.path.join(tmp_path, f"rank{i}.npz")) for i in range(p)]

    from mp_worker import problem

    w, g = problem(n, 512, k, 7)
    shards = [O.compress(g, p, s) for s in range(p)]
    w_or, v_or = w.copy(), np.zeros_like(w)
    rng = np.random.default_rng(99)
    for s in range(steps):
        x = rng.standard_normal((b, 512)).astype(np.float32)
        lab = rng.integers(0, n, b).astype(np.uint32)
        rc, loss_or, act, gf_or = O.fc_train_step_mb(w_or, v_or, x, lab, shards, m, 42, micro)
        assert rc == 0
        for r in res:
            assert abs(float(r[f"loss_{s}"]) - loss_or) <= BF16_LOSS * abs(loss_or)
        gf = np.concatenate([r[f"gf_{s}"] for r in res])
        assert rel_err(gf, gf_or) <= BF16_GRAD
    wg = np.concatenate([r["w"] for r in res])
    assert rel_err(wg - w, w_or - w) <= BF16_GRAD
    untouched = np.all(w_or == w, axis=1)
    assert np.array_equal(wg[untouched], w[untouched])


@pytest.mark.parametrize("p", [2, 4])
def test_multi_gpu_graph_ring_large_sampled(p, tmp_path):
    """The ring at 140K rows per GPU: the all-gathered pilot sample seeds the cuts and the
    candidate pass runs chunk-major over several 32K-column chunks; sampled rows bit-exact
    against build_graph_bruteforce's row (oracle), almost every row certified."""
    if _ngpus() < p:
        pytest.skip(f"needs {p} GPUs")
    n, k = 140_000 * p, 24
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={p}",
           "--master-addr=127.0.0.1", f"--master-port={29670 + p}",
           os.path.join(HERE, "mp_graph_worker.py"), "--out", str(tmp_path), "--num-classes",
           str(n), "--knn", str(k), "--ring-only"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [np.load(os.path.join(tmp_path, f"graph{i}.npz")) for i in range(p)]
    rows = np.concatenate([x["rows"] for x in res])
    assert rows.shape == (n, k)
    rc, wn, _, _ = O.l2_normalize(np.random.default_rng(5).standard_normal((n, 512)).astype(np.float32))
    assert rc == 0
    for j in np.random.default_rng(3).integers(0, n, 16):
        assert np.array_equal(rows[j], O.graph_row(wn, int(j), k)), j
    assert sum(int(x["unc"]) for x in res) < n // 1000


@pytest.mark.parametrize("p", [2, 4])
def test_multi_gpu_prepared_selection(p, tmp_path):
    """xknn_prepare over P ranks (selection collectives on the split communicator, on the side
    stream): same ActiveSets, losses and weights as the oracle."""
    if _ngpus() < p:
        pytest.skip(f"needs {p} GPUs")
    n, b, k, m, steps = 40_003, 256, 10, 4_000, 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={p}",
           "--master-addr=127.0.0.1", f"--master-port={29700 + p}",
           os.path.join(HERE, "mp_worker.py"), "--out", str(tmp_path), "--num-classes", str(n),
           "--batch", str(b), "--knn", str(k), "--m-active", str(m), "--steps", str(steps),
           "--precision", "bf16", "--prepare"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [np.load(os.path.join(tmp_path, f"rank{i}.npz")) for i in range(p)]
    from mp_worker import problem

    w, g = problem(n, 512, k, 7)
    shards = [O.compress(g, p, s) for s in range(p)]
    w_or, v_or = w.copy(), np.zeros_like(w)
    rng = np.random.default_rng(99)
    for s in range(steps):
        x = rng.standard_normal((b, 512)).astype(np.float32)
        lab = rng.integers(0, n, b).astype(np.uint32)
        rc, loss_or, act, gf_or, _ = O.fc_train_step(w_or, v_or, x, lab, shards, m, 42)
        assert rc == 0
        for r_ in res:
            assert abs(float(r_[f"loss_{s}"]) - loss_or) <= BF16_LOSS * abs(loss_or)
    wg = np.concatenate([r_["w"] for r_ in res])
    assert rel_err(wg - w, w_or - w) <= BF16_GRAD


@pytest.mark.parametrize("p", [2, 4])
def test_multi_gpu_graph_ring_and_rebuild(p, tmp_path):
    """build_graph_ring over P GPUs == build_graph_bruteforce (bit-exact rows), and the layer's
    rebuild (normalize + ring + all-to-all compression) == compress_graph(g, layout, s)."""
    if _ngpus() < p:
        pytest.skip(f"needs {p} GPUs")
    n, k = 3000, 10
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={p}",
           "--master-addr=127.0.0.1", f"--master-port={29650 + p}",
           os.path.join(HERE, "mp_graph_worker.py"), "--out", str(tmp_path), "--num-classes",
           str(n), "--knn", str(k)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = [np.load(os.path.join(tmp_path, f"graph{i}.npz")) for i in range(p)]
    from mp_graph_worker import problem

    rc, wn, _, _ = O.l2_normalize(problem(n, 5))
    assert rc == 0
    rc, g = O.bruteforce_graph("oracle", wn, k)
    assert rc == 0
    assert np.array_equal(np.concatenate([x["rows"] for x in res]), g)
    assert all(int(x["steps"]) == p - 1 for x in res)
    for s, x in enumerate(res):
        kpc, off, flat = O.compress(g, p, s)
        assert np.array_equal(x["kpc"], kpc) and np.array_equal(x["off"], off)
        assert np.array_equal(x["flat"], flat)
    # classify_retrieval over the shards: the oracle's argmax, identical on every rank
    w = problem(n, 5)
    q = np.random.default_rng(77).standard_normal((200, 512)).astype(np.float32)
    q[:3] = w[[5, n // 2, n - 1]]
    rc, want, wsc = O.classify_retrieval(q, w)
    assert rc == 0
    for x in res:
        assert np.array_equal(x["cls"], want) and np.array_equal(x["sc"], wsc)
