"""One rank of the multi-GPU parity test (launched by tests/test_gpu_multi.py under torchrun).

Every rank builds its class shard of the same seeded problem, creates an NCCL communicator
through the library's bootstrap (unique id broadcast over torch.distributed), runs selection and
fc steps, and saves its shard's results; the test compares the rank-order concatenation with the
oracle run at the same shard count P.
"""
import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))


def problem(n, d, k, seed):
    import oracle_lib as O

    rng = np.random.default_rng(seed)
    w = (rng.standard_normal((n, d)) * 0.05).astype(np.float32)
    g = O.random_graph(n, k, seed + 1)
    return w, g


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--num-classes", dest="n", type=int, default=40_000)
    ap.add_argument("--batch", dest="b", type=int, default=256)
    ap.add_argument("--knn", dest="k", type=int, default=10)
    ap.add_argument("--m-active", dest="m", type=int, default=4_000)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--precision", default="bf16")
    ap.add_argument("--prepare", action="store_true", help="pipelined selection (xknn_prepare)")
    ap.add_argument("--micro", type=int, default=1, help="StepOptions::micro_batches")
    ap.add_argument("--compact", action="store_true",
                    help="save only the changed weight rows (their local ids and deltas)")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    import paper_2102_06025_b200 as X
    from gpu_util import make_layer

    uid = [X.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = X.nccl_comm_init(uid[0], world, rank)

    n, d, b, k, m = args.n, 512, args.b, args.k, args.m
    w, g = problem(n, d, k, 7)
    prec = {"bf16": X.PREC_BF16, "fp32": X.PREC_FP32_EXACT, "fp32tc": X.PREC_FP32}[args.precision]
    layer = make_layer(n, d, world, rank, m, b, w, g, precision=prec, seed=42, comm=comm)
    rng = np.random.default_rng(99)
    bl = b // world
    res = {"begin": layer.begin, "end": layer.end}
    for s in range(args.steps):
        x = rng.standard_normal((b, d)).astype(np.float32)
        lab = rng.integers(0, n, b).astype(np.uint32)
        act, ca = layer.select_active_classes(torch.from_numpy(lab.view(np.int32)).cuda())
        res[f"active_{s}"] = act.cpu().numpy().view(np.uint32)
        res[f"contains_{s}"] = ca
        xs = torch.from_numpy(x[rank * bl:(rank + 1) * bl].copy()).cuda()
        ys = torch.from_numpy(lab[rank * bl:(rank + 1) * bl].view(np.int32).copy()).cuda()
        if args.prepare:
            layer.prepare(ys)
        gf = torch.empty(bl, d, device="cuda")
        res[f"loss_{s}"] = layer.train_step(xs, ys, 0.1, grad_features_local=gf,
                                            micro_batches=args.micro)
        res[f"gf_{s}"] = gf.cpu().numpy()
    wg = layer.weights().cpu().numpy()
    if args.compact:
        w0 = w[layer.begin:layer.end]
        rows = np.flatnonzero(np.any(wg != w0, axis=1))
        res["w_rows"] = rows.astype(np.int64)
        res["w_delta"] = wg[rows] - w0[rows]
    else:
        res["w"] = wg
    np.savez(os.path.join(args.out, f"rank{rank}.npz"), **res)
    layer.close()
    X.nccl_comm_destroy(comm)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
