"""Graph rebuild throughput (SURVEY 8d C5 reduced): xknn_graph_bruteforce on N random unit rows,
D=512.  Prints pairs/s, the GEMM-pass fraction of the bf16 peak, and uncertified rows."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2102_06025_b200 as X  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--k", type=int, default=100)
ap.add_argument("--kprime", type=int, default=0)
a = ap.parse_args()
g = torch.Generator(device="cuda")
g.manual_seed(0)
w = torch.randn(a.n, 512, device="cuda", generator=g)
w = w / w.norm(dim=1, keepdim=True)
X.graph_bruteforce(w[:4096].contiguous(), 8)  # warm-up (module load, attributes)
torch.cuda.synchronize()
t = time.perf_counter()
out, unc = X.graph_bruteforce(w, a.k, a.kprime)
torch.cuda.synchronize()
dt = time.perf_counter() - t
pairs = float(a.n) * a.n
flops = 2.0 * pairs * 512
peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))
print(json.dumps({"metric": "exact KNN graph rebuild pairs/s", "n": a.n, "k": a.k,
                  "seconds": round(dt, 3), "pairs_per_s": pairs / dt,
                  "tflops_equiv": flops / dt / 1e12,
                  "frac_of_bf16_sustained": flops / dt / 1e12 / peaks["bf16_tflops_sustained"],
                  "uncertified_rows": unc}))
