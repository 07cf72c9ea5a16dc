# C2 strong scaling on an N-GPU box: bench.py --gpus N --workload c2
N=$(nvidia-smi -L | wc -l)
mkdir -p gpurun_out
for i in 1 2; do
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2959$i bench.py --gpus $N --workload c2 --no-cpu-baseline > gpurun_out/c2_$N.json 2> gpurun_out/c2_$N.err; echo "rc=$?"
python -c "
import json;d=json.load(open('gpurun_out/c2_$N.json'));print(d['value'],d['ms_per_step'],d['e2e']['value'],{k:round(v*1000,1) for k,v in d['phase_ms'].items()})"
done
