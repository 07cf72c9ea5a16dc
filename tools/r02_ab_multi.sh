#!/bin/bash
# Bench several ab/<name> builds against the current one (fp32 C2), and a numeric comparison of
# each build's results with the current build's (relative Frobenius errors).
# usage: tools/r02_ab_multi.sh name1 name2 ...
set -u
O=gpurun_out/abm
mkdir -p $O
timeout 300 python tools/ab_bitwise.py --precision ${AB_PREC:-fp32} --save /tmp/abm_cur.pt > $O/bits_cur.txt 2>&1; echo "cur rc=$?"
for N in "$@"; do
  XKNN_PKG_DIR=ab/$N timeout 300 python tools/ab_bitwise.py --precision ${AB_PREC:-fp32} --save /tmp/abm_$N.pt > $O/bits_$N.txt 2>&1; echo "$N rc=$?"
done
python - "$@" <<'PY'
import sys, torch
c = torch.load("/tmp/abm_cur.pt")
for n in sys.argv[1:]:
    o = torch.load(f"/tmp/abm_{n}.pt")
    r = lambda a, b: float((a - b).norm() / b.norm())
    print(n, "loss rel", abs(o["loss"] - c["loss"]) / c["loss"], "gf relF", r(o["gf"], c["gf"]), "w relF", r(o["w"], c["w"]))
PY
for i in 1 2; do
  for N in cur "$@"; do
    if [ $N = cur ]; then E=""; else E="XKNN_PKG_DIR=ab/$N"; fi
    env $E timeout 300 python bench.py --precision ${AB_PREC:-fp32} --no-bf16-line --no-cpu-baseline --steps 50 --warmup 5 --e2e-steps 10 > $O/bench_${N}_$i.json 2> $O/bench_${N}_$i.err
  done
done
python - <<PY
import json,glob
for f in sorted(glob.glob("$O/bench_*.json")):
    for l in open(f):
        if l.startswith("{"):
            d=json.loads(l); print(f.split("/")[-1], d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], d["clocks"]["reasons"], {k: v for k, v in d["phase_ms"].items() if v > 0.05})
PY
