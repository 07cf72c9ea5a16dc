"""Shared helpers for the -m gpu parity tests: build a layer from host arrays, run one step."""
import numpy as np

# The stated BF16 bound: relative error of the loss, relative Frobenius error of the
# feature gradient and of the weight update, vs the fp32 reference.  Measured on B200
# (profiles/r02/parity_errors.jsonl) at C1/C2 geometries and the edge cases: loss <= 2.7e-5,
# gradients/update <= 2.5e-4 (B >= 200); a single sample carries its row's logit error whole:
# 4.9e-4 / 8.8e-4 at B = 1.  The bounds are 2x the measured maxima.
BF16_LOSS, BF16_GRAD = 6e-5, 5e-4
BF16_LOSS_B1, BF16_GRAD_B1 = 1e-3, 1.8e-3
# XKNN_PREC_FP32 (3xTF32) and FP32_EXACT: the north star's fp32 tolerance
FP32_TOL = 1e-5

import oracle_lib as O


def torch_cuda():
    import torch

    assert torch.cuda.is_available()
    return torch


def make_layer(n, d, p, rank, m, bmax, w_full, graph, *, precision, seed=42, scale=30.0,
               momentum=0.9, wd=0.0, comm=None, **kw):
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    layer = X.KnnSoftmaxLayer(n, d, rank=rank, world=p, m_active=m, max_batch=bmax, scale=scale,
                              momentum=momentum, weight_decay=wd, rng_seed=seed,
                              precision=precision, comm=comm, **kw)
    b, e = layer.begin, layer.end
    layer.set_weights(torch.from_numpy(np.ascontiguousarray(w_full[b:e])).cuda())
    kpc, off, flat = O.compress(graph, p, rank)
    layer.set_shard_graph(torch.from_numpy(kpc.view(np.int32)).cuda(),
                          torch.from_numpy(off.view(np.int64)).cuda(),
                          torch.from_numpy(flat.view(np.int32)).cuda())
    return layer


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def device_graph(n, k, seed, chunk=1 << 20):
    """A seeded self-first random k-graph generated on the device (N x k int32, row-major, as
    bench.py's install_shard_graph at P = 1): (flat, k_per_class, offsets) CUDA tensors of the
    one-shard CompressedKnnGraph.  Used where the host cannot hold the graph (C3/C4 geometry)."""
    torch = torch_cuda()
    flat = torch.empty(n * k, dtype=torch.int32, device="cuda")
    g = torch.Generator(device="cuda")
    for c0 in range(0, n, chunk):
        c1 = min(n, c0 + chunk)
        g.manual_seed(seed * 1_000_003 + c0)
        nb = torch.randint(0, n, (c1 - c0, k), device="cuda", dtype=torch.int32, generator=g)
        nb[:, 0] = torch.arange(c0, c1, device="cuda", dtype=torch.int32)
        flat[c0 * k:c1 * k] = nb.reshape(-1)
    kpc = torch.full((n,), k, dtype=torch.int32, device="cuda")
    off = torch.arange(n, device="cuda", dtype=torch.int64) * k
    return flat, kpc, off


def host_label_csr(flat_dev, n, k, labels):
    """The one-shard CSR restricted to the batch's labels (every other class gets k = 0): the
    selection reads only the labels' slices, so the oracle's result equals the full graph's."""
    torch = torch_cuda()
    u = np.unique(labels.astype(np.int64))
    rows = flat_dev.view(n, k)[torch.from_numpy(u).cuda()].cpu().numpy().view(np.uint32)
    kpc = np.zeros(n, np.uint32)
    kpc[u] = k
    off = np.zeros(n, np.uint64)
    off[1:] = np.cumsum(kpc[:-1].astype(np.uint64))
    return kpc, off, np.ascontiguousarray(rows.reshape(-1))


def parity_record(name, **vals):
    """Appends measured errors to $XKNN_PARITY_OUT (JSON lines) when set."""
    import json
    import os

    path = os.environ.get("XKNN_PARITY_OUT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"case": name, **vals}) + "\n")
    print(name, vals)
