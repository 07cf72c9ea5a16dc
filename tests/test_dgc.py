"""DGC sparsification (sparsify.cpp), the row beside the fc path: the oracle restatement of
topk_divide_conquer and CompressionState::compress_step against the compiled reference (every
chunk count, ties, multi-step residual/momentum state) and against golden vectors."""
import os

import numpy as np
import pytest

import oracle_lib as O

HERE = os.path.dirname(os.path.abspath(__file__))


def _tied(n, seed):
    rng = np.random.default_rng(seed)
    t = rng.standard_normal(n).astype(np.float32)
    t[rng.integers(0, n, n // 4)] = 0.5   # exact magnitude ties ...
    t[rng.integers(0, n, n // 8)] = -0.5  # ... across signs
    t[rng.integers(0, n, 16)] = 0.0
    t[rng.integers(0, n, 16)] = -0.0
    return t


def test_golden_topk_and_steps():
    z = np.load(os.path.join(HERE, "golden", "dgc.npz"))
    rc, idx, val = O.topk("oracle", z["t"], int(z["k"]))
    assert rc == 0 and np.array_equal(idx, z["topk_idx"]) and np.array_equal(val, z["topk_val"])
    dg = O.OracleDgc(float(z["ratio"]), float(z["momentum"]))
    for s in range(z["grads"].shape[0]):
        idx, val = dg.step(0, z["grads"][s])
        assert np.array_equal(idx, z[f"idx_{s}"]) and np.array_equal(val, z[f"val_{s}"])


def test_selected_count_kat():
    # SPEC-style: keep = ceil((1 - ratio) * len), clamped to [1, len]
    for r, n, want in [(0.999, 12345, 13), (0.0, 7, 7), (0.99, 10, 1), (0.5, 3, 2)]:
        assert O.oracle().or_selected_count(O.C.c_double(r), n) == want


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("n,k", [(5000, 1), (5000, 37), (20000, 4096), (1000, 1000)])
@pytest.mark.parametrize("chunks", [0, 1, 7, 64])
def test_topk_vs_reference(n, k, chunks):
    t = _tied(n, n + k)
    rc0, i0, v0 = O.topk("oracle", t, k)
    rc1, i1, v1 = O.topk("ref", t, k, chunks)
    assert rc0 == rc1 == 0
    assert np.array_equal(i0, i1) and np.array_equal(v0.view(np.uint32), v1.view(np.uint32))


def test_topk_errors():
    t = np.ones(10, np.float32)
    assert O.topk("oracle", t, 11)[0] != 0 and O.topk("oracle", t, 0)[0] != 0
    if O.ref_available():
        assert O.topk("ref", t, 11)[0] != 0 and O.topk("ref", t, 0)[0] != 0


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_compress_steps_vs_reference():
    rng = np.random.default_rng(3)
    ref, orc = O.RefDgc(0.99, 0.9), O.OracleDgc(0.99, 0.9)
    for step in range(6):
        for layer, n in ((0, 3000), (7, 777)):
            g = rng.standard_normal(n).astype(np.float32) * (0.1 if layer else 1.0)
            rc, i1, v1 = ref.step(layer, g, m_chunks=step)
            i0, v0 = orc.step(layer, g)
            assert rc == 0 and np.array_equal(i0, i1) and np.array_equal(v0, v1)
            assert np.array_equal(orc.state[layer][1], ref.residual(layer, n))
        if step == 3:
            assert ref.set_sparsity(0.9) == 0
            orc.ratio = 0.9
