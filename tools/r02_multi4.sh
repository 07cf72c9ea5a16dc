#!/bin/bash
# 4-GPU box: multi-GPU parity tests (P = 2, 4), then C4 (100M classes, 25M per GPU) and C3 on 4 GPUs.
O=gpurun_out
XKNN_PARITY_OUT=$O/parity_multi.jsonl timeout 1500 python -m pytest tests/test_gpu_multi.py -q -m gpu > $O/pytest_multi4.log 2>&1; echo "multi rc=$?"
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511"
timeout 1200 $R bench.py --gpus 4 --workload c4 --steps 10 --warmup 3 > $O/bench_c4_4gpu.json 2> $O/bench_c4_4gpu.err; echo "c4 rc=$?"
timeout 600 $R bench.py --gpus 4 --steps 20 --warmup 5 > $O/bench_c3_4gpu.json 2> $O/bench_c3_4gpu.err; echo "c3 rc=$?"
timeout 600 $R bench.py --gpus 4 --steps 10 --warmup 3 --precision fp32 > $O/bench_c3_4gpu_fp32.json 2> $O/bench_c3_4gpu_fp32.err; echo "c3 fp32 rc=$?"
