mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "graph" > gpurun_out/gm_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/gm_pytest.log
for C in ${CLASSES:-$((N*1000000))}; do
XKNN_GRAPH_TIMING=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 tools/bench_graph.py --classes $C --k 100 > gpurun_out/graph_${N}_$C.json 2> gpurun_out/graph_${N}_$C.err; echo "graph $C rc=$?"; grep -o '"seconds[^,]*, "pairs_per_s[^,]*,' gpurun_out/graph_${N}_$C.json; grep "candidates" gpurun_out/graph_${N}_$C.err | tail -2
done
