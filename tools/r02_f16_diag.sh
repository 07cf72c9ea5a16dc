O=gpurun_out/fdiag; mkdir -p $O
for i in 1 2; do for N in cur fnop fstg; do
  if [ $N = cur ]; then E=""; else E="XKNN_PKG_DIR=ab/$N"; fi
  env $E timeout 300 python bench.py --precision bf16 --no-bf16-line --no-cpu-baseline --steps 30 --warmup 5 --e2e-steps 5 > $O/b_${N}_$i.json 2>$O/b_${N}_$i.err
  python -c "
import json
for l in open('$O/b_${N}_$i.json'):
    if l.startswith('{'):
        d=json.loads(l); print('$N', d['ms_per_step'], d['clocks']['sm_mhz'], {k:v for k,v in d['phase_ms'].items() if v>0.03})
"
done; done
