#!/bin/bash
# ncu evidence for profiles/: the launch list of one bench run, then one --set full capture of
# the three GEMMs of one step (GEMM-F, GEMM-dW, GEMM-dX) and of the row kernels -- each only
# after the same command has exited 0 without ncu.
WL=${WL:-c2}
CMD="python bench.py --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline --workload $WL"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_full.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$WL.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_gemm2" -s 3 -c 3 -o gpurun_out/prof_${WL}_gemm $CMD > gpurun_out/ncu_full.log 2>&1
echo "full gemm rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_update_rows|k_normalize_rows" -s 3 -c 3 -o gpurun_out/prof_${WL}_rows $CMD > gpurun_out/ncu_full_rows.log 2>&1
echo "full rows rc=$?"
