#!/bin/bash
# 4-GPU box: multi-GPU parity after the batched exact top-k; C2 (the N = 1 workload) strong-
# scaled over 2 and 4 GPUs, fp32 headline + bf16 line.
O=gpurun_out/ev7
mkdir -p $O
XKNN_PARITY_OUT=$O/parity_multi.jsonl timeout 1500 python -m pytest tests/test_gpu_multi.py -q -m gpu > $O/pytest_gpu_multi_4gpu.log 2>&1; echo "multi rc=$?"; tail -1 $O/pytest_gpu_multi_4gpu.log
for N in 2 4; do
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$N"
  timeout 1200 $R bench.py --gpus $N --workload c2 --steps 20 --warmup 5 > $O/bench_c2_${N}gpu.json 2> $O/bench_c2_${N}gpu.err; echo "c2@$N rc=$?"
done
