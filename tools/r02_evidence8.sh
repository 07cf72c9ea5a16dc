#!/bin/bash
# 4-GPU box, final build: C4 (100M classes) in bf16 and C3 (fp32 + bf16) with per-rank clocks
# and phases (the softmax all-reduce wait = rank skew).
O=gpurun_out/ev8
mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 1500 $R --master-port 29581 bench.py --gpus 4 --workload c4 --precision bf16 --no-bf16-line --steps 10 --warmup 3 --e2e-steps 10 > $O/bench_c4_4gpu_bf16.json 2> $O/bench_c4_4gpu_bf16.err; echo "c4 rc=$?"
timeout 1200 $R --master-port 29582 bench.py --gpus 4 --workload c3 --steps 20 --warmup 5 > $O/bench_c3_4gpu.json 2> $O/bench_c3_4gpu.err; echo "c3 rc=$?"
