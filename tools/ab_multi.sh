# A/B of an env toggle on an N-GPU box: alternating bench.py --gpus N runs with and without it
N=$(nvidia-smi -L | wc -l)
for rep in 1 2 3; do for v in 0 1; do
  if [ $v = 1 ]; then export $AB_VAR=1; else unset $AB_VAR; fi
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2957$v bench.py --gpus $N --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "
import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$AB_VAR=$v', d['value'], d['ms_per_step'], round(d['phase_ms']['gather_normalize']*1000,1), round(d['phase_ms']['softmax_stats']*1000,1))"
done; done
