#!/bin/bash
# Round-2 evidence on one B200 (each ncu pass only after the same command exited 0 without ncu).
O=gpurun_out/ev1
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > $O/smi.txt
XKNN_PARITY_OUT=$O/parity_errors.jsonl timeout 1500 python -m pytest tests -q -m gpu > $O/pytest_gpu_1gpu.log 2>&1; echo "pytest rc=$?"
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
