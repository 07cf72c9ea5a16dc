#!/bin/bash
# Round-2 final one-B200 evidence (mixed/bf16x3 FP32 GEMMs): GPU suite with measured errors,
# smoke, the default bench line, the reference arm, C3 / C4-proxy lines per precision, the ncu
# launch list of the default command and one --set full capture per precision for the DRAM
# traffic of every step kernel (each ncu pass only after the same command exited 0 without ncu).
O=gpurun_out/ev5
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > $O/smi.txt
XKNN_PARITY_OUT=$O/parity_errors.jsonl timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu_1gpu.log 2>&1; echo "pytest rc=$?"; tail -1 $O/pytest_gpu_1gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > $O/bench_c2_default.json 2> $O/bench_c2_default.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref_c2.json 2> $O/bench_ref_c2.err; echo "ref rc=$?"
for P in fp32 bf16; do
  timeout 900 python bench.py --workload c3 --precision $P --no-bf16-line --no-cpu-baseline --steps 10 --warmup 3 > $O/bench_c3_1gpu_$P.json 2> $O/bench_c3_1gpu_$P.err; echo "c3 $P rc=$?"
  timeout 900 python bench.py --workload c4r --precision $P --no-bf16-line --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 20 > $O/bench_c4r_1gpu_$P.json 2> $O/bench_c4r_1gpu_$P.err; echo "c4r $P rc=$?"
done
CMD="python bench.py --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2_default.csv $CMD > $O/ncu_launches.log 2>&1; echo "launches rc=$?"
python tools/launch_summary.py $O/launches_c2_default.csv > $O/launches_c2_default_summary.txt 2>/dev/null
for P in fp32 bf16; do
  C="python bench.py --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-bf16-line --precision $P"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm|k_update_rows|k_normalize_rows|k_rowreduce|k_fixup|k_dx_reduce|k_zero_rows" -s 12 -c 10 -o $O/full_$P $C > $O/ncu_full_$P.log 2>&1
  echo "full $P rc=$?"
  ncu -i $O/full_$P.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,launch__grid_size > $O/full_$P.csv 2>/dev/null
  python tools/ncu_traffic.py $O/full_$P.csv > $O/traffic_c2_$P.json
done
ls -la $O | head -40
