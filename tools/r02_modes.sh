#!/bin/bash
# FP32 GEMM arithmetic modes (XKNN_FP32_GEMM = mixed | f3 | 3xtf32): fp32 parity tests with the
# measured errors recorded per mode, then alternating C2 bench lines.
# usage: tools/r02_modes.sh "<modes to test>" "<modes to bench>"
set -u
O=gpurun_out/modes
mkdir -p $O
for M in $1; do
  XKNN_FP32_GEMM=$M XKNN_PARITY_OUT=$O/parity_$M.jsonl timeout 900 python -m pytest tests -m gpu -x -q -k "fp32tc or tensor_cores or shim or free_func" > $O/pytest_$M.log 2>&1; echo "pytest $M rc=$?"; tail -1 $O/pytest_$M.log
done
for i in 1 2; do
  for M in $2; do
    XKNN_FP32_GEMM=$M timeout 300 python bench.py --precision fp32 --no-bf16-line --no-cpu-baseline --steps 50 --warmup 5 --e2e-steps 20 > $O/bench_${M}_$i.json 2> $O/bench_${M}_$i.err
  done
done
python - <<PY
import json,glob
for f in sorted(glob.glob("$O/bench_*.json")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f.split("/")[-1], d["value"], d["ms_per_step"], d["e2e"]["value"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], {k: v for k, v in d["phase_ms"].items() if v > 0.05})
PY
python - <<PY
import json,glob
for f in sorted(glob.glob("$O/parity_*.jsonl")):
    for l in open(f):
        r=json.loads(l)
        if "steps" in r: r={"case":r["case"],"gf":max(s["gf_relF"] for s in r["steps"]),"update_relF":r["update_relF"],"velocity_relF":r["velocity_relF"],"loss":max(s["loss_rel"] for s in r["steps"])}
        print(f.split("/")[-1], r["case"], {k: "%.2e" % v for k, v in r.items() if isinstance(v, float)})
PY
