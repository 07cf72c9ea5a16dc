#!/bin/bash
# 4-GPU box, final build: the default workload (C2) on 2 and 4 GPUs -- the driver's scaling
# configuration -- with per-rank clocks and phases.
O=gpurun_out/ev9
mkdir -p $O
for N in 2 4; do
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$N"
  timeout 1200 $R bench.py --gpus $N --steps 30 --warmup 5 > $O/bench_c2_${N}gpu.json 2> $O/bench_c2_${N}gpu.err; echo "c2@$N rc=$?"
done
