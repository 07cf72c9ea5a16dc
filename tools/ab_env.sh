# Same-box comparison of environment settings (ENVS="A=1 B=2;C=3", ';'-separated variants,
# an empty variant = baseline) on bench.py --gpus N (N = visible GPUs)
N=$(nvidia-smi -L | wc -l)
IFS=';' read -ra VARS <<< "$ENVS"
for rep in 1 2; do i=0; for v in "${VARS[@]}"; do i=$((i+1))
  env $v timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2958$i bench.py --gpus $N --no-cpu-baseline > gpurun_out/ae_$i.json 2> gpurun_out/ae_$i.err
  python -c "
import json;d=json.load(open('gpurun_out/ae_$i.json'));p=d['phase_ms'];print('[$v]', d['value'], d['ms_per_step'], round(p['softmax_stats']*1000,1), round(p['dX_reduce_scatter']*1000,1), round(p['update']*1000,1))"
done; done
