#!/bin/bash
# One ncu --set full capture of each hot kernel (GEMM-F/dW/dX pair kernels, row update, gather)
# after the same command has exited 0 without ncu; plus the launch list.
WL=${WL:-c2}
CMD="python bench.py --steps 3 --warmup 1 --no-cpu-baseline --workload $WL"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_full.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$WL.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_gemm2|k_update_rows|k_normalize_rows" -s 4 -c 5 -o gpurun_out/prof_$WL $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
