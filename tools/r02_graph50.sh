#!/bin/bash
# C5 upper end on a 4-GPU box: the ring build at 50M classes (12.5M rows per GPU), k = 100,
# k' = 200, clocks sampled, 16 sampled rows verified bit-exact against the oracle.
O=gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531"
XKNN_GRAPH_TIMING=1 timeout 3000 $R tools/bench_graph.py --classes 50000000 --k 100 --kprime 200 --verify 16 > $O/graph_50m_4gpu.json 2> $O/graph_50m_4gpu.err
echo "graph50 rc=$?"
