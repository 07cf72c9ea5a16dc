"""DGC on device (dgc.cu) vs the oracle restatement (tests/test_dgc.py pins it to the reference):
exact top-k indices/values (bit-exact, ties and signed zeros included) and multi-layer,
multi-step compress_step outputs plus residual/velocity state."""
import numpy as np
import pytest

import oracle_lib as O
from gpu_util import torch_cuda
from test_dgc import _tied

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,k", [(1, 1), (5000, 1), (5000, 37), (200_000, 4096), (3000, 3000)])
def test_topk_device(n, k):
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    t = _tied(n, n + k) if n > 1 else np.array([-2.5], np.float32)
    idx, val = X.topk(torch.from_numpy(t).cuda(), k)
    rc, i0, v0 = O.topk("oracle", t, k)
    assert rc == 0
    assert np.array_equal(idx.cpu().numpy().astype(np.uint64), i0)
    assert np.array_equal(val.cpu().numpy().view(np.uint32), v0.view(np.uint32))


def test_topk_device_errors():
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    t = torch.ones(10, device="cuda")
    with pytest.raises(X.KTooLarge):
        X.topk(t, 11)
    with pytest.raises(X.InvalidArgument):
        X.topk(t, 0)


def test_compress_steps_device():
    import paper_2102_06025_b200 as X

    torch = torch_cuda()
    rng = np.random.default_rng(5)
    dev, orc = X.CompressionState(0.99, 0.9), O.OracleDgc(0.99, 0.9)
    for step in range(5):
        for layer, n in ((0, 100_000), (3, 777), (9, 1)):
            g = rng.standard_normal(n).astype(np.float32)
            if step == 2:
                g[: n // 2] = 0.0  # ties in the residual
            i1, v1 = dev.compress_step(layer, torch.from_numpy(g).cuda())
            i0, v0 = orc.step(layer, g)
            assert np.array_equal(i1.cpu().numpy().astype(np.uint64), i0), (step, layer)
            assert np.array_equal(v1.cpu().numpy(), v0)
            r, v = dev.state(layer, n)
            assert np.array_equal(r.cpu().numpy(), orc.state[layer][1])
            assert np.array_equal(v.cpu().numpy(), orc.state[layer][0])
        if step == 2:
            dev.set_sparsity_ratio(0.9)
            orc.ratio = 0.9
    with pytest.raises(X.ShapeMismatch):
        dev.compress_step(3, torch.zeros(778, device="cuda"))
    with pytest.raises(X.InvalidArgument):
        dev.compress_step(4, torch.zeros(0, device="cuda"))
    with pytest.raises(X.InvalidArgument):
        X.CompressionState(1.0, 0.9)
    dev.close()
