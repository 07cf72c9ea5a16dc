#!/bin/bash
# bf16x3 backward GEMMs: parity (fp32 tests, measured errors recorded), bitwise-independent
# A/B of XKNN_FP32_BWD=tf32 vs the default, bench lines for both.
set -u
O=gpurun_out/bf3
mkdir -p $O
XKNN_PARITY_OUT=$O/parity_bf3.jsonl timeout 900 python -m pytest tests -m gpu -x -q -k "fp32tc or tensor_cores or shim or free_func" > $O/pytest_bf3.log 2>&1; echo "pytest bf3 rc=$?"; tail -3 $O/pytest_bf3.log
XKNN_FP32_BWD=tf32 XKNN_PARITY_OUT=$O/parity_tf32.jsonl timeout 900 python -m pytest tests -m gpu -x -q -k "fp32tc or tensor_cores" > $O/pytest_tf32.log 2>&1; echo "pytest tf32 rc=$?"; tail -1 $O/pytest_tf32.log
for i in 1 2; do
  timeout 300 python bench.py --precision fp32 --no-bf16-line --no-cpu-baseline --steps 50 --warmup 5 --e2e-steps 20 > $O/bench_bf3_$i.json 2> $O/bench_bf3_$i.err
  XKNN_FP32_BWD=tf32 timeout 300 python bench.py --precision fp32 --no-bf16-line --no-cpu-baseline --steps 50 --warmup 5 --e2e-steps 20 > $O/bench_tf32_$i.json 2> $O/bench_tf32_$i.err
done
python - <<PY
import json,glob
for f in sorted(glob.glob("$O/bench_*.json")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f.split("/")[-1], d["value"], d["ms_per_step"], d["e2e"]["value"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], {k: v for k, v in d["phase_ms"].items() if v > 0.05})
PY
