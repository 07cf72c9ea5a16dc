#!/bin/bash
# Final one-B200 check of the shipped build: GPU suite (measured errors), smoke, the default
# bench line and the reference arm.
O=gpurun_out/final1
mkdir -p $O
XKNN_PARITY_OUT=$O/parity_errors.jsonl timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu_1gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu_1gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$? $(cat $O/smoke.log | tail -1)"
timeout 900 python bench.py > $O/bench_c2_default.json 2> $O/bench_c2_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref_c2.json 2> $O/bench_ref_c2.err; echo "ref rc=$?"
python - <<PY
import json
for f in ["$O/bench_c2_default.json", "$O/bench_ref_c2.json"]:
    for l in open(f):
        if l.startswith("{"):
            d = json.loads(l)
            print(f.split("/")[-1], d.get("value"), d.get("ms_per_step"), d.get("e2e", {}).get("value"), d.get("clocks", {}).get("sm_mhz"), (d.get("bf16_mode") or {}).get("value"))
PY
