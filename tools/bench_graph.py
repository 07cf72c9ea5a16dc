"""KNN class-graph rebuild throughput (BASELINE config 5): xknn_graph_ring over
P GPUs (one process per GPU; torchrun for P > 1) on N synthetic class weights, D = 512.

    python tools/bench_graph.py --n 1000000 --k 100
    torchrun --nproc-per-node 2 tools/bench_graph.py --n 4000000 --k 100

Prints one JSON line: pairs/s (N^2 / time, max over ranks), the candidate GEMM's tensor-core
work as a fraction of the measured bf16/fp16 peak, uncertified rows.  Weights are random
N(0, 1) rows normalized on device (random-init class weights, as the bench's fc layer)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("XKNN_PKG_DIR"):  # A/B runs against another build of the package
    sys.path.insert(0, os.environ["XKNN_PKG_DIR"])
import torch  # noqa: E402

import paper_2102_06025_b200 as X  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--classes", type=int, default=1_000_000)
ap.add_argument("--k", type=int, default=100)
ap.add_argument("--kprime", type=int, default=200)
a = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
comm = None
if world > 1:
    import torch.distributed as dist

    dist.init_process_group("gloo")
    uid = [X.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = X.nccl_comm_init(uid[0], world, rank)
b, e = X.ShardLayout(a.classes, world).class_range(rank)
g = torch.Generator(device="cuda")
g.manual_seed(1000 + rank)
w = torch.empty(e - b, 512, device="cuda")
for r0 in range(0, e - b, 1 << 20):
    blk = torch.randn(min(1 << 20, e - b - r0), 512, device="cuda", generator=g)
    w[r0:r0 + blk.shape[0]] = blk / blk.norm(dim=1, keepdim=True)
    del blk
# warm-up (module load, kernel attributes, NCCL channels) on a small problem
ws = w[: max(64, min(4096, e - b))].contiguous()
X.graph_ring(ws, ws.shape[0] * world if world > 1 else ws.shape[0], 8, 16, rank, world, comm) \
    if world == 1 else None
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
# two full-size builds; the second is timed (the first pays the allocator's first touches)
for rep in range(2):
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    out, unc, steps = X.graph_ring(w, a.classes, a.k, a.kprime, rank, world, comm)
    ev1.record()
    ev1.synchronize()
    sec = ev0.elapsed_time(ev1) / 1e3
    del out
if world > 1:
    t = torch.tensor([sec, float(unc)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sec = float(t[0])
    ut = torch.tensor([float(unc)], dtype=torch.float64)
    dist.all_reduce(ut)
    unc = int(ut.item())
if rank == 0:
    peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))
    pairs = float(a.classes) * a.classes
    tf = 2.0 * pairs * 512 / sec / 1e12
    print(json.dumps({"metric": "exact KNN graph rebuild pairs/s", "n": a.classes, "k": a.k,
                      "kprime": a.kprime, "n_gpus": world, "seconds": round(sec, 3),
                      "pairs_per_s": pairs / sec, "tflops_equiv": round(tf, 1),
                      "frac_of_tensor_peak": round(tf / (world * peaks["bf16_tflops_sustained"]), 4),
                      "peak_source": "MEASURED_PEAKS bf16 sustained (fp16 same rate)",
                      "uncertified_rows": unc, "transfer_steps": int(steps)}))
if world > 1:
    X.nccl_comm_destroy(comm)
    dist.destroy_process_group()
