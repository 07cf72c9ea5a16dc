#!/bin/bash
# ncu --set full of one fp32 step's GEMMs + normalize + update (after a clean run), CSV raw page.
set -u
O=gpurun_out/prof_fp32
mkdir -p $O
CMD="python bench.py --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-bf16-line --precision fp32"
timeout 300 $CMD > $O/plain.log 2>&1 || { echo plain failed; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm3" -s 3 -c 3 -o $O/full $CMD > $O/ncu.log 2>&1
echo "ncu rc=$?"
ncu -i $O/full.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
ncu -i $O/full.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
