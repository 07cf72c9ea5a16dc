import sys, os, time
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch
import oracle_lib as O
from gpu_util import make_layer, rel_err
import paper_2102_06025_b200 as X
n, d, b, k, m = 20_000, 512, 256, 10, 2_000
rng = np.random.default_rng(0)
w = (rng.standard_normal((n, d)) * 0.05).astype(np.float32)
g = O.random_graph(n, k, 1); sh = [O.compress(g, 1, 0)]
for prec in (X.PREC_FP32, X.PREC_BF16):
    L = make_layer(n, d, 1, 0, m, b, w, g, precision=prec)
    wo, vo = w.copy(), np.zeros_like(w)
    for s in range(2):
        x = rng.standard_normal((b, d)).astype(np.float32); lab = rng.integers(0, n, b).astype(np.uint32)
        rc, lo, act, gfo, _ = O.fc_train_step(wo, vo, x, lab, sh, m, 42)
        gf = torch.empty(b, d, device="cuda")
        l = L.train_step(torch.from_numpy(x).cuda(), torch.from_numpy(lab.view(np.int32)).cuda(), 0.1, grad_features_local=gf)
        print(f"prec={prec} step {s}: loss {l:.9f} oracle {lo:.9f} rel {abs(l-lo)/lo:.2e} gf relF {rel_err(gf.cpu().numpy(), gfo):.2e}", flush=True)
    wg = L.weights().cpu().numpy()
    print(f"  upd relF {rel_err(wg-w, wo-w):.2e}", flush=True)
    L.close()
