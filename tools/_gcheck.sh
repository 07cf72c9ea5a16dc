mkdir -p gpurun_out
for rep in 1 2; do for v in 0 1; do
  if [ $v = 1 ]; then export XKNN_NO_PILOT=1; else unset XKNN_NO_PILOT; fi
  XKNN_GCHUNK=256 XKNN_GRAPH_TIMING=1 timeout 300 python tools/bench_graph.py --classes 1000000 --k 100 > gpurun_out/gc_$v.json 2> gpurun_out/gc_$v.err; echo "nopilot=$v rc=$? $(grep -o '"seconds[^,]*,' gpurun_out/gc_$v.json)"; tail -4 gpurun_out/gc_$v.err
done; done
