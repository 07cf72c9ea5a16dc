#!/bin/bash
# quick experiment: bf16 step parity + bench (in-kernel and separate update)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_step.py -x -q -k bf16 > gpurun_out/exp_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/exp_pytest.log
for f in "" "--separate-update"; do
timeout 300 python bench.py --no-cpu-baseline --steps 20 $f > gpurun_out/exp_bench.json 2>gpurun_out/exp_bench.err; echo "bench $f rc=$?"
python -c "import json;d=json.load(open('gpurun_out/exp_bench.json'));print(d['value'],d['ms_per_step'],d['phase_ms'])" || tail -5 gpurun_out/exp_bench.err
done
