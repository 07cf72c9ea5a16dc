"""Shared helpers for the -m gpu parity tests: build a layer from host arrays, run one step."""
import numpy as np

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
