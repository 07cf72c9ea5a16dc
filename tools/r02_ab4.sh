O=gpurun_out/ab4; mkdir -p $O
for i in 1 2; do for N in cur ovl0; do
  if [ $N = cur ]; then E=""; else E="XKNN_PKG_DIR=ab/$N"; fi
  env $E timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2959$i bench.py --gpus 4 --workload c2 --steps 30 --warmup 5 --e2e-steps 30 --no-cpu-baseline --bf16-pause 3 > $O/b_${N}_$i.json 2> $O/b_${N}_$i.err
  python - <<PY
import json
for l in open("$O/b_${N}_$i.json"):
    if l.startswith("{"):
        d=json.loads(l); b=d.get("bf16_mode") or {}
        print("$N", "fp32", d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], "bf16", b.get("value"), b.get("ms_per_step"))
PY
done; done
