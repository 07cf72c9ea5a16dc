mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_graph.py -x -q > gpurun_out/gg_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/gg_pytest.log
for c in 0.16 0.14; do
  XKNN_NO_PILOT=1 XKNN_GRAPH_SCAN_ONLY=$c XKNN_GCHUNK=256 timeout 300 python tools/bench_graph.py --classes 1000000 --k 100 > /dev/null 2> gpurun_out/gs_$c.err; grep "scan only" gpurun_out/gs_$c.err | tail -1
done
for rep in 1 2; do for v in 0 1; do
  if [ $v = 1 ]; then export XKNN_NO_PILOT=1; else unset XKNN_NO_PILOT; fi
  XKNN_GCHUNK=256 XKNN_GRAPH_TIMING=1 timeout 300 python tools/bench_graph.py --classes 1000000 --k 100 > gpurun_out/gc_$v.json 2> gpurun_out/gc_$v.err; echo "nopilot=$v rc=$? $(grep -o '"seconds[^,]*,' gpurun_out/gc_$v.json) $(grep -o 'candidates.*pilot [0-9.]*' gpurun_out/gc_$v.err | tail -1) $(grep -o 'uncertified [0-9]*' gpurun_out/gc_$v.err | tail -1)"
done; done
