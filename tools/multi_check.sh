mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/gm_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/gm_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus $N > gpurun_out/bench_c3_$N.json 2> gpurun_out/bench_c3_$N.err; echo "bench rc=$? size=$(wc -c < gpurun_out/bench_c3_$N.json)"; grep '^{' gpurun_out/bench_c3_$N.json | python -c "
import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],d['e2e']['value'],d['roofline']['kernel'],d['roofline']['frac'],{k:round(v*1000,1) for k,v in d['phase_ms'].items()})"
