#!/bin/bash
# ncu evidence for profiles/: launch list of one bench run + one --set full capture of the GEMMs.
CMD="python bench.py --steps 3 --warmup 1 --no-cpu-baseline --workload c2"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 3 -c 3 -o gpurun_out/prof_gemm $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
$CMD > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_update_rows|k_normalize_rows" -s 2 -c 2 -o gpurun_out/prof_rows $CMD > gpurun_out/ncu_rows.log 2>&1
echo "rows rc=$?"
