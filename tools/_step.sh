mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_step.py -x -q > gpurun_out/gs_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/gs_pytest.log
for i in 1 2 3; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err; echo "bench rc=$?"; python -c "
import json;d=json.load(open('gpurun_out/bench_s.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],d['gpu_launches'])"; done
