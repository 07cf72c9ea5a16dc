mkdir -p gpurun_out
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err; echo "bench rc=$?"; python -c "
import json;d=json.load(open('gpurun_out/bench_s.json'));print(d['value'],d['ms_per_step'],d['e2e'])"; done
