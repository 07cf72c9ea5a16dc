#!/bin/bash
# Round-2 evidence on a 4-GPU box: multi-GPU parity (P = 2, 4), C3 on 2 and 4 GPUs (fp32 headline
# + bf16 line) with the mixed/bf16x3 FP32 GEMMs.
O=gpurun_out/ev6
mkdir -p $O
XKNN_PARITY_OUT=$O/parity_multi.jsonl timeout 1500 python -m pytest tests/test_gpu_multi.py -q -m gpu > $O/pytest_gpu_multi_4gpu.log 2>&1; echo "multi rc=$?"
for N in 2 4; do
  R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$N"
  timeout 1200 $R bench.py --gpus $N --steps 20 --warmup 5 > $O/bench_c3_${N}gpu.json 2> $O/bench_c3_${N}gpu.err; echo "c3@$N rc=$?"
done
