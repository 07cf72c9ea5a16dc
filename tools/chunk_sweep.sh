for rep in 1 2; do for c in ${CHUNKS:-128 256 512}; do
XKNN_GCHUNK=$c XKNN_GRAPH_TIMING=1 timeout 300 python tools/bench_graph.py --classes 1000000 --k 100 > gpurun_out/gk_$c.json 2> gpurun_out/gk_$c.err; echo "chunk=$c $(grep -o '"seconds[^,]*,' gpurun_out/gk_$c.json) $(grep -o 'candidates [0-9.]*' gpurun_out/gk_$c.err | tail -1)"
done; done
