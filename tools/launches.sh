#!/bin/bash
# bench run + its ncu launch list (per-kernel device times, serialized / cold-cache)
CMD="python bench.py --steps 3 --warmup 1 --no-cpu-baseline --workload ${WL:-c2}"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${WL:-c2}.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
