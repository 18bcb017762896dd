N=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29540 bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/bench_n$N.json 2> /dev/null
python -c "
import json; d=json.load(open('gpurun_out/bench_n$N.json')); print(d['ms_per_step'], d['parity'], d['e2e'])"
timeout 600 python -m pytest tests/test_gpu_summa.py -x -q -m gpu -k "gather or e2e or 1x2" 2>&1 | tail -2
