#!/bin/bash
# One --set full capture of a step's three GEMMs (and the row update) on workload $WL, precision
# $P, after the same command exited 0 without ncu; raw metrics exported to CSV.
WL=${WL:-c2}; P=${P:-bf16}; O=gpurun_out; TAG=${TAG:-$WL_$P}
CMD="python bench.py --steps 2 --warmup 1 --e2e-steps 1 --no-cpu-baseline --workload $WL --precision $P"
timeout 900 $CMD > $O/plain_$TAG.log 2>&1 || { echo "plain $TAG failed"; exit 1; }
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k_gemm|k_update_rows" -s 8 -c 4 -o $O/full_$TAG $CMD > $O/ncu_full_$TAG.log 2>&1
echo "full $TAG rc=$?"
ncu -i $O/full_$TAG.ncu-rep --page raw --csv > $O/full_${TAG}_raw.csv 2>/dev/null
ncu -i $O/full_$TAG.ncu-rep --page details --csv > $O/full_${TAG}_details.csv 2>/dev/null
python tools/ncu_traffic.py $O/full_${TAG}_raw.csv > $O/traffic_$TAG.json
