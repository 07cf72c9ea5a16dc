"""One fc train step on device vs the oracle restatement of HybridSim::train_step's fc half
(bit-exact with the reference, tests/test_oracle.py).

FP32_EXACT: logits bit-identical (same summation order, no FMA); loss, weights, velocity and
feature gradients within 1e-5 relative (CUDA expf vs glibc expf, NCCL/parallel reduction order).
FP32 (tensor cores at fp32 accuracy, fast32.cu): 1e-5 relative, as FP32_EXACT.
BF16: tensor-core GEMMs with bf16 operands; the stated bound (gpu_util.BF16_*) is
6e-5 relative on the loss and 5e-4 relative (Frobenius) on the weight update and the feature
gradient (1e-3 / 1.8e-3 for a single-sample batch): twice the measured maxima.
"""
import numpy as np
import pytest

import oracle_lib as O
from gpu_util import (BF16_GRAD, BF16_GRAD_B1, BF16_LOSS, BF16_LOSS_B1, make_layer,
                      parity_record, rel_err, torch_cuda)

pytestmark = pytest.mark.gpu


def _run(n, d, b, k, m, precision, steps=2, seed=42, lr=0.1, wd=0.0, check_logits=False, **kw):
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    rng = np.random.default_rng(n + b)
    w = (rng.standard_normal((n, d)) * 0.05).astype(np.float32)
    g = O.random_graph(n, k, 3)
    shards = [O.compress(g, 1, 0)]
    layer = make_layer(n, d, 1, 0, m, b, w, g, precision=precision, seed=seed, wd=wd, **kw)
    w_or, v_or = w.copy(), np.zeros_like(w)
    out = []
    for step in range(steps):
        x = rng.standard_normal((b, d)).astype(np.float32)
        lab = rng.integers(0, n, b).astype(np.uint32)
        rc, loss_or, act, gf_or, logits_or = O.fc_train_step(w_or, v_or, x, lab, shards, m, seed,
                                                             lr=lr, wd=wd,
                                                             want_logits=check_logits)
        assert rc == 0
        gf = torch.empty(b, d, device="cuda")
        loss = layer.train_step(torch.from_numpy(x).cuda(),
                                torch.from_numpy(lab.view(np.int32)).cuda(), lr,
                                grad_features_local=gf)
        if check_logits:
            lg = layer.last_logits(b)
            assert lg.shape == logits_or.shape
            if step == 0:  # identical inputs: identical fp32 logits (reference summation order)
                assert np.array_equal(lg, logits_or), np.abs(lg - logits_or).max()
            else:  # weights now carry the (tolerance-level) update difference
                assert rel_err(lg, logits_or) <= 1e-5
        out.append(dict(loss=loss, loss_or=loss_or, gf=gf.cpu().numpy(), gf_or=gf_or))
    wg = layer.weights().cpu().numpy()
    vg = layer.velocity().cpu().numpy()
    layer.close()
    return out, wg, w_or, vg, v_or, w


@pytest.mark.parametrize("n,b,k,m", [(20_000, 128, 10, 2_000), (12_000, 64, 20, 500)])
def test_step_fp32_exact(n, b, k, m):
    import paper_2102_06025_b200 as X

    out, wg, w_or, vg, v_or, w0 = _run(n, 512, b, k, m, X.PREC_FP32_EXACT, steps=3,
                                       check_logits=True)
    for o in out:
        assert abs(o["loss"] - o["loss_or"]) <= 1e-5 * abs(o["loss_or"])
        assert rel_err(o["gf"], o["gf_or"]) <= 1e-5
    assert rel_err(wg - w0, w_or - w0) <= 1e-5  # the update itself
    assert rel_err(vg, v_or) <= 1e-5
    untouched = np.all(w_or == w0, axis=1)  # non-active rows unchanged
    assert np.array_equal(wg[untouched], w0[untouched])


def test_step_fp32_exact_weight_decay():
    import paper_2102_06025_b200 as X

    out, wg, w_or, vg, v_or, w0 = _run(8_000, 256, 32, 8, 800, X.PREC_FP32_EXACT, steps=2,
                                       wd=1e-3)
    assert rel_err(wg - w0, w_or - w0) <= 1e-5
    for o in out:
        assert abs(o["loss"] - o["loss_or"]) <= 1e-5 * abs(o["loss_or"])


def _errors(out, wg, w_or, vg, v_or, w0):
    upd, upd_or = wg - w0, w_or - w0
    return dict(loss_rel=max(abs(o["loss"] - o["loss_or"]) / abs(o["loss_or"]) for o in out),
                gf_relF=max(rel_err(o["gf"], o["gf_or"]) for o in out),
                update_relF=rel_err(upd, upd_or), velocity_relF=rel_err(vg, v_or))


SHAPES = [(100_000, 256, 10, 10_000), (20_000, 512, 10, 2_000), (30_000, 200, 10, 3_001)]
EDGES = [(9_000, 1, 10, 150),       # one sample, M_w < one tile
         (50_000, 1024, 12, 2_000), # over-full ranking branch
         (70_001, 333, 7, 7_001),   # ragged batch and class tiles
         (30_000, 4_500, 10, 6_000)]  # > 16 batch row tiles, ragged (GEMM-dX split-K units)


@pytest.mark.parametrize("n,b,k,m", SHAPES + EDGES)
def test_step_fp32_tensor_cores(n, b, k, m):
    """XKNN_PREC_FP32 (tcgen05 GEMMs at fp32 accuracy: mixed tf32/bf16 logits, bf16x3 gradients):
    the north star's fp32 tolerance, 1e-5 relative, on the loss, the feature gradient, the
    weight update and the velocity."""
    import paper_2102_06025_b200 as X

    out, wg, w_or, vg, v_or, w0 = _run(n, 512, b, k, m, X.PREC_FP32, steps=3, wd=1e-4)
    e = _errors(out, wg, w_or, vg, v_or, w0)
    parity_record(f"fp32tc_{n}_{b}_{k}_{m}", **e)
    assert e["loss_rel"] <= 1e-5, e
    assert e["gf_relF"] <= 1e-5, e
    assert e["update_relF"] <= 1e-5, e
    assert e["velocity_relF"] <= 1e-5, e
    untouched = np.all(w_or == w0, axis=1)
    assert np.array_equal(wg[untouched], w0[untouched])


@pytest.mark.parametrize("n,b,k,m", SHAPES)
def test_step_bf16(n, b, k, m):
    import paper_2102_06025_b200 as X

    out, wg, w_or, vg, v_or, w0 = _run(n, 512, b, k, m, X.PREC_BF16, steps=2, wd=1e-4)
    parity_record(f"bf16_{n}_{b}_{k}_{m}", **_errors(out, wg, w_or, vg, v_or, w0))
    for o in out:
        assert abs(o["loss"] - o["loss_or"]) <= BF16_LOSS * abs(o["loss_or"]), (o["loss"], o["loss_or"])
        assert rel_err(o["gf"], o["gf_or"]) <= BF16_GRAD
    assert rel_err(wg - w0, w_or - w0) <= BF16_GRAD
    untouched = np.all(w_or == w0, axis=1)
    assert np.array_equal(wg[untouched], w0[untouched])


@pytest.mark.parametrize("n,b,k,m", EDGES)
def test_step_bf16_edges(n, b, k, m):
    import paper_2102_06025_b200 as X

    out, wg, w_or, vg, v_or, w0 = _run(n, 512, b, k, m, X.PREC_BF16, steps=3)
    parity_record(f"bf16_{n}_{b}_{k}_{m}", **_errors(out, wg, w_or, vg, v_or, w0))
    # the per-row bf16 logit error (~1e-4 of s per cosine) averages over the batch; a single
    # sample carries it whole (gpu_util.BF16_*_B1)
    tol, tg = (BF16_LOSS_B1, BF16_GRAD_B1) if b == 1 else (BF16_LOSS, BF16_GRAD)
    for o in out:
        assert abs(o["loss"] - o["loss_or"]) <= tol * abs(o["loss_or"]), (o["loss"], o["loss_or"])
        assert rel_err(o["gf"], o["gf_or"]) <= tg
    assert rel_err(wg - w0, w_or - w0) <= tg
    untouched = np.all(w_or == w0, axis=1)
    assert np.array_equal(wg[untouched], w0[untouched])


@pytest.mark.parametrize("precision", ["bf16", "fp32", "fp32tc"])
def test_step_errors_leave_parameters(precision):
    """LabelOutOfRange / MTooSmall surface at sync with the reference's error class, and the
    step touches no parameter (the reference throws before the update)."""
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    prec = {"bf16": X.PREC_BF16, "fp32": X.PREC_FP32_EXACT, "fp32tc": X.PREC_FP32}[precision]
    n, b, k = 6_000, 64, 5
    rng = np.random.default_rng(1)
    w = (rng.standard_normal((n, 512)) * 0.05).astype(np.float32)
    g = O.random_graph(n, k, 2)
    layer = make_layer(n, 512, 1, 0, 600, b, w, g, precision=prec, seed=42)
    x = torch.from_numpy(rng.standard_normal((b, 512)).astype(np.float32)).cuda()
    lab = rng.integers(0, n, b).astype(np.int32)
    bad = lab.copy()
    bad[17] = n + 5
    with pytest.raises(X.LabelOutOfRange):
        layer.train_step(x, torch.from_numpy(bad).cuda(), 0.1)
    assert np.array_equal(layer.weights().cpu().numpy(), w)
    # M smaller than the number of distinct labels
    small = make_layer(n, 512, 1, 0, 10, b, w, g, precision=prec, seed=42)
    with pytest.raises(X.MTooSmall):
        small.train_step(x, torch.from_numpy(lab).cuda(), 0.1)
    assert np.array_equal(small.weights().cpu().numpy(), w)
    # the layer recovers: a valid step afterwards matches the oracle
    loss = layer.train_step(x, torch.from_numpy(lab).cuda(), 0.1)
    w_or, v_or = w.copy(), np.zeros_like(w)
    rc, loss_or, _, _, _ = O.fc_train_step(w_or, v_or, x.cpu().numpy(), lab.view(np.uint32),
                                          [O.compress(g, 1, 0)], 600, 42)
    assert rc == 0
    tol = BF16_LOSS if precision == "bf16" else 1e-5
    assert abs(loss - loss_or) <= tol * abs(loss_or)
    layer.close()
    small.close()


@pytest.mark.parametrize("precision", ["bf16", "fp32", "fp32tc"])
def test_step_with_prepared_selection(precision):
    """xknn_prepare: the next step's selection runs on the side stream while the current step is
    in flight; results equal the oracle's (and the unprepared path), including steps that are not
    prepared and a prepared selection superseded by xknn_select."""
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    prec = {"bf16": X.PREC_BF16, "fp32": X.PREC_FP32_EXACT, "fp32tc": X.PREC_FP32}[precision]
    n, b, k, m = 30_000, 256, 10, 3_000
    rng = np.random.default_rng(4)
    w = (rng.standard_normal((n, 512)) * 0.05).astype(np.float32)
    g = O.random_graph(n, k, 6)
    shards = [O.compress(g, 1, 0)]
    layer = make_layer(n, 512, 1, 0, m, b, w, g, precision=prec, seed=42)
    xs = [rng.standard_normal((b, 512)).astype(np.float32) for _ in range(6)]
    labs = [rng.integers(0, n, b).astype(np.uint32) for _ in range(6)]
    dev_lab = [torch.from_numpy(l.view(np.int32)).cuda() for l in labs]
    w_or, v_or = w.copy(), np.zeros_like(w)
    plan = [True, True, False, True, True, True]  # step 2 runs its own selection
    layer.prepare(dev_lab[0])
    for s in range(6):
        if s == 4:  # a superseded prepare: xknn_select in between, then prepare again
            got, _ = layer.select_active_classes(dev_lab[s])
            rc, want, _ = O.select_shards("oracle", n, shards, labs[s], m, 42)
            assert rc == 0 and np.array_equal(got.cpu().numpy().view(np.uint32), want)
            layer.prepare(dev_lab[s])
        layer.train_step(torch.from_numpy(xs[s]).cuda(), dev_lab[s], 0.1, sync=False)
        if s + 1 < 6 and plan[s + 1]:
            layer.prepare(dev_lab[s + 1])
        layer.sync()
        loss = float(layer._loss.item())
        rc, loss_or, act, _, _ = O.fc_train_step(w_or, v_or, xs[s], labs[s], shards, m, 42)
        assert rc == 0
        tol = BF16_LOSS if precision == "bf16" else 1e-5
        assert abs(loss - loss_or) <= tol * abs(loss_or), (s, loss, loss_or)
        t, l = layer.last_active()
        assert l == act.size
    wg = layer.weights().cpu().numpy()
    assert rel_err(wg - w, w_or - w) <= (BF16_GRAD if precision == "bf16" else 1e-5)
    layer.close()


@pytest.mark.parametrize("precision,micro,b", [("fp32", 2, 64), ("fp32", 3, 50), ("bf16", 4, 256),
                                               ("bf16", 7, 100), ("fp32tc", 3, 300)])
def test_step_micro_batches(precision, micro, b):
    """StepOptions::micro_batches (parallel.cpp:444, :505-591) through xknn_step_micro against the
    oracle's micro-batch step (bit-exact with the stock HybridSim, tests/test_oracle.py): loss,
    weights, velocity, and the per-micro-batch feature gradient handed to mlp_backward."""
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    prec = {"bf16": X.PREC_BF16, "fp32": X.PREC_FP32_EXACT, "fp32tc": X.PREC_FP32}[precision]
    tol_l, tol_g = (BF16_LOSS, BF16_GRAD) if precision == "bf16" else (1e-5, 1e-5)
    n, d, k, m, seed = 20_000, 512, 10, 2_000, 42
    rng = np.random.default_rng(micro + b)
    w = (rng.standard_normal((n, d)) * 0.05).astype(np.float32)
    g = O.random_graph(n, k, 3)
    shards = [O.compress(g, 1, 0)]
    layer = make_layer(n, d, 1, 0, m, b, w, g, precision=prec, seed=seed)
    w_or, v_or = w.copy(), np.zeros_like(w)
    for _ in range(2):
        x = rng.standard_normal((b, d)).astype(np.float32)
        lab = rng.integers(0, n, b).astype(np.uint32)
        rc, loss_or, act, gf_or = O.fc_train_step_mb(w_or, v_or, x, lab, shards, m, seed, micro)
        assert rc == 0
        gf = torch.empty(b, d, device="cuda")
        loss = layer.train_step(torch.from_numpy(x).cuda(),
                                torch.from_numpy(lab.view(np.int32)).cuda(), 0.1,
                                grad_features_local=gf, micro_batches=micro)
        assert abs(loss - loss_or) <= tol_l * abs(loss_or), (loss, loss_or)
        gfn = gf.cpu().numpy()
        assert rel_err(gfn, gf_or) <= tol_g
        # per micro-batch too: each carries its own 1/m_c
        base, rem = divmod(b, micro)
        off = 0
        for c in range(micro):
            rc_ = base + (1 if c < rem else 0)
            assert rel_err(gfn[off:off + rc_], gf_or[off:off + rc_]) <= tol_g
            off += rc_
    wg = layer.weights().cpu().numpy()
    vg = layer.velocity().cpu().numpy()
    layer.close()
    assert rel_err(wg - w, w_or - w) <= tol_g
    assert rel_err(vg, v_or) <= tol_g
    untouched = np.all(w_or == w, axis=1)
    assert np.array_equal(wg[untouched], w[untouched])


def test_step_loss_into_pinned_host_memory():
    """train_step's loss written straight into pinned host memory (the e2e loop's path) equals
    the device-memory loss of the same step."""
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    n, b, k, m = 20_000, 128, 10, 2_000
    rng = np.random.default_rng(8)
    w = (rng.standard_normal((n, 512)) * 0.05).astype(np.float32)
    g = O.random_graph(n, k, 3)
    x = torch.from_numpy(rng.standard_normal((b, 512)).astype(np.float32)).cuda()
    lab = torch.from_numpy(rng.integers(0, n, b).astype(np.int32)).cuda()
    out = []
    for dest in ("cuda", "pinned"):
        layer = make_layer(n, 512, 1, 0, m, b, w, g, precision=X.PREC_BF16, seed=42)
        buf = (torch.zeros(1, dtype=torch.float64, device="cuda") if dest == "cuda"
               else torch.zeros(1, dtype=torch.float64).pin_memory())
        layer.train_step(x, lab, 0.1, loss_out=buf, sync=False)
        layer.sync()
        out.append(float(buf.cpu()[0]))
        layer.close()
    assert out[0] == out[1] and np.isfinite(out[0]) and out[0] > 0


@pytest.mark.parametrize("precision", ["bf16", "fp32tc"])
def test_step_active_capacity_exceeded(precision):
    """xknn_config_t::active_capacity below the shard's active count: the step fails with
    OutOfMemory at sync and touches no parameter; a layer with room runs the same step."""
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    prec = {"bf16": X.PREC_BF16, "fp32tc": X.PREC_FP32}[precision]
    n, b, k, m = 20_000, 128, 10, 2_000
    rng = np.random.default_rng(3)
    w = (rng.standard_normal((n, 512)) * 0.05).astype(np.float32)
    g = O.random_graph(n, k, 2)
    x = torch.from_numpy(rng.standard_normal((b, 512)).astype(np.float32)).cuda()
    lab = torch.from_numpy(rng.integers(0, n, b).astype(np.int32)).cuda()
    small = make_layer(n, 512, 1, 0, m, b, w, g, precision=prec, seed=42, active_capacity=1_500)
    with pytest.raises(X.OutOfMemory):
        small.train_step(x, lab, 0.1)
    assert np.array_equal(small.weights().cpu().numpy(), w)
    roomy = make_layer(n, 512, 1, 0, m, b, w, g, precision=prec, seed=42, active_capacity=2_000)
    loss = roomy.train_step(x, lab, 0.1)
    assert np.isfinite(loss)
    small.close()
    roomy.close()


@pytest.mark.parametrize("mode", ["mixed", "f3", "3xtf32", "bogus"])
def test_fp32_gemm_modes(mode, monkeypatch):
    """XKNN_FP32_GEMM selects the FP32 path's GEMM arithmetic; every mode meets the fp32 bar on
    a small step (the full parity suite runs on the default), an unknown one is a ConfigError."""
    import paper_2102_06025_b200 as X

    monkeypatch.setenv("XKNN_FP32_GEMM", mode)
    if mode == "bogus":
        with pytest.raises(X.ConfigError):
            X.KnnSoftmaxLayer(1000, 512, m_active=100, max_batch=8, precision=X.PREC_FP32)
        return
    out, wg, w_or, vg, v_or, w0 = _run(20_000, 512, 256, 10, 2_000, X.PREC_FP32, steps=2)
    e = _errors(out, wg, w_or, vg, v_or, w0)
    assert max(e.values()) <= 1e-5, e
