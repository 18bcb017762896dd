N=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/bn$N.json 2> gpurun_out/bn$N.log
echo rc=$?; tail -3 gpurun_out/bn$N.log; python -c "
import json; d=json.load(open('gpurun_out/bn$N.json')); print({k: d.get(k) for k in ('value','ms_per_step','parity')}, d['roofline']['frac'], d['config']['threshold_bytes'], d['e2e'])"
