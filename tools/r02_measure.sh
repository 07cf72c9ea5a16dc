#!/bin/bash
# Round-2 evidence in one gpurun call (1 GPU): TF32 peak, the two precisions' bench lines, the
# ncu launch list and one --set full capture of a step's kernels per precision (each only after
# the same command exited 0 without ncu), exported to CSV for tools/ncu_traffic.py.
set -u
O=gpurun_out
mkdir -p $O
timeout 120 python tools/measure_tf32.py > $O/tf32_peak.json 2> $O/tf32.err; echo "tf32 rc=$?"
for P in bf16 fp32; do
  CMD="python bench.py --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline --precision $P"
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --precision $P > $O/bench_$P.json 2> $O/bench_$P.err
  echo "bench $P rc=$?"
  timeout 300 $CMD > $O/plain_$P.log 2>&1 || { echo "plain $P failed"; continue; }
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$P.csv $CMD > $O/ncu_launches_$P.log 2>&1
  echo "launches $P rc=$?"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm|k_update_rows|k_normalize_rows" -s 12 -c 6 -o $O/full_$P $CMD > $O/ncu_full_$P.log 2>&1
  echo "full $P rc=$?"
  ncu -i $O/full_$P.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,sm__throughput.avg.pct_of_peak_sustained_elapsed > $O/full_$P.csv 2>/dev/null
  python tools/ncu_traffic.py $O/full_$P.csv > $O/traffic_c2_$P.json
done
