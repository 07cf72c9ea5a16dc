# C3 on one GPU: the three GEMMs of one step under ncu --set full (after a plain run)
CMD="python bench.py --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline --workload c3"
mkdir -p gpurun_out
timeout 900 $CMD > gpurun_out/plain_c3.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain_c3.log; exit 1; }
grep '^{' gpurun_out/plain_c3.log | python -c "
import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],{k:round(v*1000,1) for k,v in d['phase_ms'].items()})"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_gemm2" -s 3 -c 3 -o gpurun_out/prof_c3_gemm $CMD > gpurun_out/ncu_c3.log 2>&1
echo "ncu rc=$?"
