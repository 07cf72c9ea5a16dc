set -u
O=gpurun_out/prof3
mkdir -p $O
CMD="python bench.py --steps 3 --warmup 1 --e2e-steps 1 --no-cpu-baseline --no-bf16-line --precision fp32"
timeout 300 $CMD > $O/plain.log 2>&1 || { echo plain failed; exit 1; }
for V in cur pconv0; do
  if [ $V = cur ]; then E=""; else E="XKNN_PKG_DIR=ab/$V"; fi
  env $E timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm3" -s 3 -c 3 -o $O/full_$V $CMD > $O/ncu_$V.log 2>&1
  echo "ncu $V rc=$?"
  ncu -i $O/full_$V.ncu-rep --page raw --csv > $O/raw_$V.csv 2>/dev/null
  ncu -i $O/full_$V.ncu-rep --page details --csv > $O/details_$V.csv 2>/dev/null
done
ls -la $O
