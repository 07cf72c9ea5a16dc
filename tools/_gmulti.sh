mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/gm_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/gm_pytest.log
XKNN_GRAPH_TIMING=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 tools/bench_graph.py --classes $((N*1000000)) --k 100 > gpurun_out/graph_$N.json 2> gpurun_out/graph_$N.err; echo "graph rc=$?"; cat gpurun_out/graph_$N.json; grep "candidates" gpurun_out/graph_$N.err | tail -2
