"""One rank of the multi-GPU graph-rebuild parity test (launched by tests/test_gpu_multi.py):
xknn_graph_ring on this rank's normalized block, and xknn_layer_rebuild_graph on the live layer
(normalize + ring + all-to-all compression); results saved for comparison with the oracle."""
import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(HERE))


def problem(n, seed):
    rng = np.random.default_rng(seed)
    nb = n // 10
    base = rng.standard_normal((nb, 512)).astype(np.float32)
    w = np.concatenate([base, base, base + 1e-4 * rng.standard_normal((nb, 512)).astype(np.float32),
                        rng.standard_normal((n - 3 * nb, 512)).astype(np.float32)])
    return (w[rng.permutation(n)] * 0.05).astype(np.float32)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", required=True)
    ap.add_argument("--num-classes", dest="n", type=int, default=3000)
    ap.add_argument("--knn", dest="k", type=int, default=10)
    ap.add_argument("--ring-only", action="store_true",
                    help="random unit rows, graph_ring only (large-n runs checked on sampled rows)")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("gloo")
    import oracle_lib as O
    import paper_2102_06025_b200 as X

    uid = [X.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    comm = X.nccl_comm_init(uid[0], world, rank)
    n, k = args.n, args.k
    w = (np.random.default_rng(5).standard_normal((n, 512)).astype(np.float32) if args.ring_only
         else problem(n, 5))
    rc, wn, _, _ = O.l2_normalize(w)
    assert rc == 0
    b, e = O.shard_range(n, world, rank)
    rows, unc, steps = X.graph_ring(torch.from_numpy(np.ascontiguousarray(wn[b:e])).cuda(), n, k,
                                    2 * k, rank, world, comm)
    if args.ring_only:
        np.savez(os.path.join(args.out, f"graph{rank}.npz"),
                 rows=rows.cpu().numpy().view(np.uint32), unc=unc, steps=steps)
        X.nccl_comm_destroy(comm)
        dist.barrier()
        dist.destroy_process_group()
        return
    layer = X.KnnSoftmaxLayer(n, 512, rank=rank, world=world, m_active=n // 10, max_batch=64,
                              rng_seed=42, comm=comm)
    layer.set_weights(torch.from_numpy(np.ascontiguousarray(w[b:e])).cuda())
    unc2 = layer.rebuild_graph(k)
    kpc, off, flat = layer.graph()
    q = np.random.default_rng(77).standard_normal((200, 512)).astype(np.float32)
    q[:3] = w[[5, n // 2, n - 1]]
    cls, sc = layer.classify(torch.from_numpy(q).cuda())
    np.savez(os.path.join(args.out, f"graph{rank}.npz"), rows=rows.cpu().numpy().view(np.uint32),
             unc=unc, unc2=unc2, steps=steps, kpc=kpc, off=off, flat=flat,
             cls=cls.cpu().numpy().view(np.uint32), sc=sc.cpu().numpy())
    layer.close()
    X.nccl_comm_destroy(comm)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
