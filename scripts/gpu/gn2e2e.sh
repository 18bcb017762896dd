N=$(nvidia-smi -L | wc -l)
for f in 0.1 1.0; do
SPG_D2H_GPU_WIDEN=$f timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29540 bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/n${N}_e2e_$f.json 2> /dev/null
python -c "
import json; d=json.load(open('gpurun_out/n${N}_e2e_$f.json')); print('$f', d['ms_per_step'], d['parity'], d['e2e']['seconds'])"
done
