"""One train step of a small layer (bring-up / fault isolation; XKNN_DEBUG_SYNC=1 reports a
faulting kernel at its launch site; XKNN_PKG_DIR=<dir> runs another build).
usage: python tools/step_small.py N B M [bf16|fp32|fp32_exact]"""
import os, sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
if os.environ.get("XKNN_PKG_DIR"):
    sys.path.insert(0, os.environ["XKNN_PKG_DIR"])
import numpy as np, torch
import oracle_lib as O
from gpu_util import make_layer
import paper_2102_06025_b200 as X
n, d, b, k, m = int(sys.argv[1]), 512, int(sys.argv[2]), 10, int(sys.argv[3])
rng = np.random.default_rng(0)
w = (rng.standard_normal((n, d)) * 0.05).astype(np.float32)
g = O.random_graph(n, k, 1)
prec = {'bf16': X.PREC_BF16, 'fp32': X.PREC_FP32, 'fp32_exact': X.PREC_FP32_EXACT}[sys.argv[4] if len(sys.argv) > 4 else 'bf16']
L = make_layer(n, d, 1, 0, m, b, w, g, precision=prec)
x = rng.standard_normal((b, d)).astype(np.float32); lab = rng.integers(0, n, b).astype(np.uint32)
gf = torch.empty(b, d, device="cuda")
l = L.train_step(torch.from_numpy(x).cuda(), torch.from_numpy(lab.view(np.int32)).cuda(), 0.1, grad_features_local=gf)
print("loss", l, X.__file__)
