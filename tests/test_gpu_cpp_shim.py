"""The C++ drop-in shim (include/xcls_gpu.hpp) driven by a compiled C++ caller
(tests/cpp/shim_caller.cpp, written against the reference's xcls:: API) on the GPU, against the
oracle: select_active_classes over the full KnnGraph and over P compressed shards (bit-exact),
knn_softmax_forward_backward (1e-5), two HybridSim fc steps with P simulated workers' graphs in
XKNN_PREC_FP32 (1e-5), and the reference's exception classes."""
import os
import subprocess

import numpy as np
import pytest

import oracle_lib as O
from gpu_util import rel_err
from test_abi import compile_shim_caller

pytestmark = pytest.mark.gpu


def test_cpp_caller_vs_oracle(tmp_path):
    n, k, b, d, m, seed, p = 30_000, 10, 210, 512, 3_000, 42, 3  # B % P == 0 (HybridSim)
    rng = np.random.default_rng(12)
    g = O.random_graph(n, k, 5)
    lab = rng.integers(0, n, b).astype(np.uint32)
    _, xn, _, _ = O.l2_normalize(rng.standard_normal((b, d)).astype(np.float32))
    _, wn, _, _ = O.l2_normalize(rng.standard_normal((n, d)).astype(np.float32))
    wraw = (rng.standard_normal((n, d)) * 0.05).astype(np.float32)
    feat = rng.standard_normal((b, d)).astype(np.float32)
    t = tmp_path
    np.array([n, k, b, d, m, seed, p], np.uint64).tofile(t / "meta.bin")
    for name, a in (("graph", g), ("labels", lab), ("xnorm", xn), ("wnorm", wn), ("wraw", wraw),
                    ("feat", feat)):
        np.ascontiguousarray(a).tofile(t / f"{name}.bin")
    exe = str(t / "shim_caller")
    compile_shim_caller(exe)
    r = subprocess.run([exe, str(t)], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]

    rc, want_full, _ = O.select_full("oracle", g, lab, m, seed)
    assert rc == 0
    assert np.array_equal(np.fromfile(t / "sel_full.bin", np.uint32), want_full)
    shards = [O.compress(g, p, s) for s in range(p)]
    rc, want_span, _ = O.select_shards("oracle", n, shards, lab, m, seed)
    assert rc == 0
    act = np.fromfile(t / "sel_span.bin", np.uint32)
    assert np.array_equal(act, want_span)

    rc, loss_or, _, gf_or, gw_or = O.knn_softmax_fwd_bwd("oracle", xn, wn, lab, act, 30.0)
    assert rc == 0
    loss = float(np.fromfile(t / "fb_loss.bin", np.float64)[0])
    assert abs(loss - loss_or) <= 1e-5 * abs(loss_or)
    assert rel_err(np.fromfile(t / "fb_gf.bin", np.float32).reshape(b, d), gf_or) <= 1e-5
    gw = np.fromfile(t / "fb_gw.bin", np.float32).reshape(n, d)
    assert rel_err(gw[act.astype(np.int64)], gw_or) <= 1e-5
    mask = np.ones(n, bool)
    mask[act.astype(np.int64)] = False
    assert not gw[mask].any()  # dense grad_weights: exactly zero outside the active rows

    w_or, v_or = wraw.copy(), np.zeros_like(wraw)
    losses = np.fromfile(t / "sim_loss.bin", np.float64)
    for s in range(2):
        rc, l_or, _, gf_or, _ = O.fc_train_step(w_or, v_or, feat, lab, shards, m, seed)
        assert rc == 0
        assert abs(losses[s] - l_or) <= 1e-5 * abs(l_or)
    assert rel_err(np.fromfile(t / "sim_gf.bin", np.float32).reshape(b, d), gf_or) <= 1e-5
    wt = np.fromfile(t / "sim_w.bin", np.float32).reshape(n, d)
    assert rel_err(wt - wraw, w_or - wraw) <= 1e-5
    assert int(np.fromfile(t / "errs.bin", np.int32)[0]) == 7
