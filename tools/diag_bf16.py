"""Diagnostic: BF16 and FP32_EXACT step errors vs the oracle, plus a rough C2 step time."""
import sys, time, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import oracle_lib as O
from gpu_util import make_layer, rel_err
import paper_2102_06025_b200 as X

def run(n, d, b, k, m, prec, steps=2):
    rng = np.random.default_rng(1)
    w = (rng.standard_normal((n, d)) * 0.05).astype(np.float32)
    g = O.random_graph(n, k, 3); sh = [O.compress(g, 1, 0)]
    L = make_layer(n, d, 1, 0, m, b, w, g, precision=prec)
    wo, vo = w.copy(), np.zeros_like(w)
    for s in range(steps):
        x = rng.standard_normal((b, d)).astype(np.float32); lab = rng.integers(0, n, b).astype(np.uint32)
        rc, lo, act, gfo, _ = O.fc_train_step(wo, vo, x, lab, sh, m, 42)
        gf = torch.empty(b, d, device="cuda")
        l = L.train_step(torch.from_numpy(x).cuda(), torch.from_numpy(lab.view(np.int32)).cuda(), 0.1, grad_features_local=gf)
        print(f"  prec={prec} step {s}: loss {l:.9f} oracle {lo:.9f} rel {abs(l-lo)/lo:.2e}  gf relF {rel_err(gf.cpu().numpy(), gfo):.2e}")
    wg = L.weights().cpu().numpy()
    print(f"  dW relF {rel_err(wg-w, wo-w):.2e}  maxabs {np.abs((wg-w)-(wo-w)).max():.2e} / {np.abs(wo-w).max():.2e}")
    L.close()

print("C1-like N=100K B=256 k=10 M=10K")
run(100_000, 512, 256, 10, 10_000, X.PREC_BF16)
run(100_000, 512, 256, 10, 10_000, X.PREC_FP32_EXACT)
print("N=20K B=1000 (ragged batch) M=3000")
run(20_000, 512, 1000, 10, 3_000, X.PREC_BF16)
# rough C2 timing
n, b, k, m = 1_000_000, 1024, 50, 100_000
L = X.KnnSoftmaxLayer(n, 512, m_active=m, max_batch=b, rng_seed=42, precision=X.PREC_BF16)
L.weights_view().tensor.normal_(0, 0.05)
gr = torch.randint(0, n, (n, k), device="cuda", dtype=torch.int32); gr[:, 0] = torch.arange(n, device="cuda", dtype=torch.int32)
kpc = torch.full((n,), k, dtype=torch.int32, device="cuda"); off = torch.arange(n, device="cuda", dtype=torch.int64) * k
L.set_shard_graph(kpc, off, gr.reshape(-1))
xs = torch.randn(b, 512, device="cuda"); ls = torch.randint(0, n, (b,), device="cuda", dtype=torch.int32)
for i in range(3): L.train_step(xs, ls, 0.1)
torch.cuda.synchronize(); t = time.time()
for i in range(20): L.train_step(xs, ls, 0.1, sync=False)
torch.cuda.synchronize(); dt = (time.time() - t) / 20
L.sync()
print(f"C2 step {dt*1e3:.3f} ms -> {b/dt:.0f} samples/s ; launches {L.kernel_launches}")
