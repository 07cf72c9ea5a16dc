"""Bitwise A/B of two builds of the package on one workload: runs `--steps` train steps (bench.py's
synthetic C2 data) and prints the loss bits, a checksum of d loss / d features and checksums of
the weight and velocity shards.  Run once plain and once with XKNN_PKG_DIR=<other build>; equal
lines mean the two builds compute identical results.
usage: python tools/ab_bitwise.py [--workload c2] [--precision fp32] [--steps 3]"""
import argparse
import os
import struct
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
if os.environ.get("XKNN_PKG_DIR"):
    sys.path.insert(0, os.environ["XKNN_PKG_DIR"])

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2102_06025_b200 as X  # noqa: E402


def checksum(t):
    v = t.contiguous().view(torch.int32).to(torch.int64).flatten()
    w = torch.arange(1, v.numel() + 1, device=v.device, dtype=torch.int64) % 1000003
    return int(v.sum().item()), int((v * w).sum().item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--save", default="", help="torch.save the last d loss / d features and the "
                    "weight rows that changed, for a numeric comparison of builds that differ")
    a = ap.parse_args()
    wl = bench.WORKLOADS[a.workload]
    n, b, k = wl["n"], wl["b"], wl["k"]
    m = max(1, (n + 9) // 10)
    prec = {"bf16": X.PREC_BF16, "fp32": X.PREC_FP32, "fp32_exact": X.PREC_FP32_EXACT}[a.precision]
    torch.cuda.set_device(0)
    layer = X.KnnSoftmaxLayer(n, bench.D, m_active=m, max_batch=b, scale=bench.SCALE,
                              momentum=bench.MOMENTUM, rng_seed=bench.SEED, precision=prec)
    gw = torch.Generator(device="cuda")
    gw.manual_seed(10)
    wv = layer.weights_view().tensor
    for r0 in range(0, wv.shape[0], 1 << 20):
        wv[r0:r0 + (1 << 20)].normal_(0.0, 0.05, generator=gw)
    bench.install_shard_graph(torch, layer, n, k, 1, 0)
    batches = bench.make_batches(torch, n, b, 0)
    gf = torch.empty(b, bench.D, device="cuda")
    w0 = layer.weights_view().tensor[: 1 << 15].clone()
    print("lib", X.__file__)
    for s in range(a.steps):
        x, y = batches[s % len(batches)]
        loss = layer.train_step(x, y, bench.LR, grad_features_local=gf)
        torch.cuda.synchronize()
        print(f"step {s} loss {loss!r} bits {struct.pack('<d', loss).hex()} gf {checksum(gf)}")
    W = layer.weights_view().tensor
    print("W", checksum(W), "V", checksum(layer.velocity()))
    if a.save:
        torch.save({"gf": gf.cpu(), "w": (W[: 1 << 15] - w0).cpu(), "loss": loss}, a.save)


if __name__ == "__main__":
    main()
