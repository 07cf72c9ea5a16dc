"""XKNN graph files (save_graph / load_graph, knn_graph.cpp:276-311) through the library's
row-distributed I/O (xknn_graph_save_rows / xknn_graph_load_rows): byte-identical to the
reference's writer (golden file from oracle/_ref, tests/golden/make_golden.py), the reference's
error classes, and shards of a ShardLayout writing one file from separate processes (gloo)."""
import os

import numpy as np
import pytest

import oracle_lib as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "graph_small.xknn")


def _x():
    import paper_2102_06025_b200 as X

    return X


def test_save_is_byte_identical_to_reference(tmp_path):
    X = _x()
    g = O.random_graph(50, 5, 31)  # the graph make_golden.py saved with the reference
    p = str(tmp_path / "g.xknn")
    X.save_graph_rows(p, 50, 0, g, create=True)
    assert open(p, "rb").read() == open(GOLDEN, "rb").read()


def test_load_reference_file():
    X = _x()
    k, rows = X.load_graph_rows(GOLDEN, 50)
    assert k == 5 and np.array_equal(rows, O.random_graph(50, 5, 31))
    k, part = X.load_graph_rows(GOLDEN, 50, 17, 33)
    assert np.array_equal(part, rows[17:33])


@pytest.mark.parametrize("p", [2, 3, 7])
def test_shards_write_one_file(tmp_path, p):
    X = _x()
    g = O.random_graph(50, 5, 31)
    path = str(tmp_path / "g.xknn")
    order = [0] + list(range(p - 1, 0, -1))  # header writer first, the rest in any order
    for s in order:
        b, e = O.shard_range(50, p, s)
        X.save_graph_rows(path, 50, b, g[b:e], create=(s == 0))
    assert open(path, "rb").read() == open(GOLDEN, "rb").read()
    for s in range(p):
        b, e = O.shard_range(50, p, s)
        assert np.array_equal(X.load_graph_rows(path, 50, b, e)[1], g[b:e])


def _bytes_with(mutate):
    data = bytearray(open(GOLDEN, "rb").read())
    return bytes(mutate(data))


@pytest.mark.parametrize("case,exc", [
    ("magic", "IoError"), ("version", "IoError"), ("trunc_header", "IoError"),
    ("trunc_body", "IoError"), ("k_varies", "IoError"), ("classes", "ShapeMismatch"),
    ("missing", "IoError"),
])
def test_load_errors(tmp_path, case, exc):
    X = _x()
    path = str(tmp_path / "bad.xknn")

    def mut(d):
        if case == "magic":
            d[0:4] = b"XKNM"
        elif case == "version":
            d[4] = 2
        elif case == "trunc_header":
            d = d[:12]
        elif case == "trunc_body":
            d = d[:-3]
        elif case == "k_varies":
            d[16 + 24 * 7] = 4  # class 7's k
        return d

    if case != "missing":
        open(path, "wb").write(_bytes_with(mut))
    n = 51 if case == "classes" else 50
    with pytest.raises(getattr(X, exc)):
        X.load_graph_rows(path, n)
    if O.ref_available() and case not in ("classes", "missing"):
        rc, _ = O.ref_load_graph(path)  # the reference rejects the same files
        assert rc != 0


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_roundtrip_with_reference(tmp_path):
    X = _x()
    g = O.random_graph(1000, 13, 4)
    a, b = str(tmp_path / "a.xknn"), str(tmp_path / "b.xknn")
    assert O.ref_save_graph(a, g) == 0
    k, rows = X.load_graph_rows(a, 1000)
    assert k == 13 and np.array_equal(rows, g)
    X.save_graph_rows(b, 1000, 0, g, create=True)
    rc, back = O.ref_load_graph(b)
    assert rc == 0 and np.array_equal(back, g)


def _gloo_rank(rank, world, port, path, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X = _x()
    n, k = 1000, 13
    g = O.random_graph(n, k, 4)
    b, e = X.ShardLayout(n, world).class_range(rank)
    if rank == 0:
        X.save_graph_rows(path, n, b, g[b:e], create=True)
    dist.barrier()
    if rank != 0:
        X.save_graph_rows(path, n, b, g[b:e], create=False)
    dist.barrier()
    kk, rows = X.load_graph_rows(path, n, b, e)
    np.save(os.path.join(out, f"r{rank}.npy"), rows)
    dist.destroy_process_group()


def test_gloo_two_ranks_share_one_file(tmp_path):
    """Two processes, one shard each: rank 0 writes the header and its rows, rank 1 its rows;
    each reads its rows back; the file equals the reference writer's output."""
    import torch.multiprocessing as mp

    path = str(tmp_path / "g.xknn")
    port = 29400 + os.getpid() % 500
    mp.spawn(_gloo_rank, args=(2, port, path, str(tmp_path)), nprocs=2, join=True)
    g = O.random_graph(1000, 13, 4)
    rows = np.concatenate([np.load(str(tmp_path / f"r{r}.npy")) for r in range(2)])
    assert np.array_equal(rows, g)
    if O.ref_available():
        rc, back = O.ref_load_graph(path)
        assert rc == 0 and np.array_equal(back, g)
