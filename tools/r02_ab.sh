#!/bin/bash
# One-GPU A/B of the current build against ab/<name> (tools/ab_build.sh): bitwise results
# (tools/ab_bitwise.py), the fp32 GPU tests, and alternating bench lines.
# usage: tools/r02_ab.sh <name> [precision] [tests -k expr]
set -u
NAME=$1; P=${2:-fp32}; K=${3:-fp32}
O=gpurun_out/ab_$NAME
mkdir -p $O
timeout 300 python tools/ab_bitwise.py --precision $P > $O/bits_new.txt 2> $O/bits_new.err; echo "bits new rc=$?"
XKNN_PKG_DIR=ab/$NAME timeout 300 python tools/ab_bitwise.py --precision $P > $O/bits_old.txt 2> $O/bits_old.err; echo "bits old rc=$?"
if diff <(grep -v ^lib $O/bits_new.txt) <(grep -v ^lib $O/bits_old.txt) > /dev/null; then echo "BITWISE IDENTICAL"; else echo "BITWISE DIFFER"; fi
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > $O/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.log
for i in 1 2; do
  timeout 300 python bench.py --precision $P --no-bf16-line --no-cpu-baseline --steps 50 --warmup 5 --e2e-steps 20 > $O/bench_new_$i.json 2> $O/bench_new_$i.err
  XKNN_PKG_DIR=ab/$NAME timeout 300 python bench.py --precision $P --no-bf16-line --no-cpu-baseline --steps 50 --warmup 5 --e2e-steps 20 > $O/bench_old_$i.json 2> $O/bench_old_$i.err
done
python - <<PY
import json,glob
for f in sorted(glob.glob("$O/bench_*.json")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f.split("/")[-1], d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], {k: v for k, v in d["phase_ms"].items() if v > 0.05})
PY
