bash tools/r02_ab_multi.sh fmkb16
O=gpurun_out/prof_dx
mkdir -p $O
CMD="python bench.py --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-bf16-line --precision fp32"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm3<3>" -s 1 -c 1 -o $O/full $CMD > $O/ncu.log 2>&1
echo "ncu rc=$?"
ncu -i $O/full.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
