"""Generates tests/golden/*.npz from the COMPILED REFERENCE (oracle/_ref/libxcls_ref.so, built by
`make -C oracle ref` from /root/reference/proj/src).  Run in the build container:

    python tests/golden/make_golden.py

The fixtures pin the C restatement in oracle/ on machines where /root/reference is absent.
Inputs are regenerated from the recorded seeds by tests/oracle_lib.random_graph / numpy.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_lib as O  # noqa: E402


def selection_cases():
    cases = []
    # (n, k, b, p, m, seed, graph_seed, label_seed): padding, exact-fit and over-full branches,
    # including the C1 geometry (N=100K, B=256, k=10, M=10% of N).
    specs = [
        (100_000, 10, 256, 1, 10_000, 42, 11, 21),
        (100_000, 10, 256, 1, 1_000, 42, 11, 22),
        (100_000, 10, 256, 8, 1_000, 42, 11, 23),
        (20_000, 10, 256, 2, 2_000, 7, 12, 24),
        (20_000, 10, 256, 4, 400, 7, 12, 25),
        (5_000, 50, 64, 4, 500, 99, 13, 26),
        (5_000, 50, 64, 8, 3_000, 3, 13, 27),
        (1_000, 12, 100, 1, 100, 1, 14, 28),
        (1_000, 12, 10, 2, 1_000, 5, 14, 29),  # M == N: every class
    ]
    for n, k, b, p, m, seed, gs, ls in specs:
        g = O.random_graph(n, k, gs)
        lab = np.random.default_rng(ls).integers(0, n, b).astype(np.uint32)
        shards = [O.compress(g, p, s) for s in range(p)]
        rc, act, ca = O.select_shards("ref", n, shards, lab, m, seed)
        assert rc == 0
        cases.append(dict(n=n, k=k, b=b, p=p, m=m, seed=seed, graph_seed=gs, labels=lab,
                          active=act, contains_all=ca))
    return cases


def step_case():
    n, d, b, k, m, p = 1500, 64, 32, 6, 150, 2
    rng = np.random.default_rng(5)
    w = (rng.standard_normal((n, d)) * 0.05).astype(np.float32)
    g = O.random_graph(n, k, 15)
    shards = [O.compress(g, p, s) for s in range(p)]
    sim = O.RefSim(w, p)
    sim.set_graphs(shards)
    xs, ls, losses, ws = [], [], [], []
    for _ in range(2):
        x = rng.standard_normal((b, d)).astype(np.float32)
        lab = rng.integers(0, n, b).astype(np.uint32)
        rc, loss, _ = sim.step(x, lab, m, 42)
        assert rc == 0
        xs.append(x)
        ls.append(lab)
        losses.append(loss)
    ws = sim.weights()
    return dict(n=n, d=d, b=b, k=k, m=m, p=p, graph_seed=15, w_seed=5, x=np.stack(xs),
                labels=np.stack(ls), losses=np.array(losses), w_final=ws)


def main():
    assert O.ref_available(), "build oracle/_ref first: make -C oracle ref"
    for i, c in enumerate(selection_cases()):
        np.savez_compressed(os.path.join(HERE, f"select_{i}.npz"), **c)
    np.savez_compressed(os.path.join(HERE, "fc_step.npz"), **step_case())
    rng = np.random.default_rng(3)
    w = rng.standard_normal((300, 16)).astype(np.float32)
    _, wn, _, _ = O.l2_normalize(w)
    rc, gr = O.bruteforce_graph("ref", wn, 7)
    assert rc == 0
    np.savez_compressed(os.path.join(HERE, "graph_bf.npz"), w=w, k=7, graph=gr)
    # an XKNN graph file written by the reference's save_graph (knn_graph.cpp:276-291)
    g = O.random_graph(50, 5, 31)
    assert O.ref_save_graph(os.path.join(HERE, "graph_small.xknn"), g) == 0
    # DGC: topk_divide_conquer and three compress_step calls of the reference
    rng = np.random.default_rng(11)
    t = rng.standard_normal(3000).astype(np.float32)
    t[rng.integers(0, 3000, 500)] = 0.25
    rc, i, v = O.topk("ref", t, 100, 5)
    assert rc == 0
    grads = np.stack([rng.standard_normal(2000).astype(np.float32) for _ in range(3)])
    dg, out = O.RefDgc(0.98, 0.9), {}
    for s in range(3):
        rc, ii, vv = dg.step(0, grads[s])
        assert rc == 0
        out[f"idx_{s}"], out[f"val_{s}"] = ii, vv
    np.savez_compressed(os.path.join(HERE, "dgc.npz"), t=t, k=100, topk_idx=i, topk_val=v,
                        ratio=0.98, momentum=0.9, grads=grads, **out)


if __name__ == "__main__":
    main()
