# final sweep on N GPUs: config-2 bench line, configs 3-5 lines (parity vs oracle goldens)
N=$(nvidia-smi -L | wc -l)
if [ "$N" = 1 ]; then
  timeout 900 python bench.py > gpurun_out/sweep_c2_n1.json 2> gpurun_out/sweep_c2_n1.log; echo c2 rc=$?
else
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29540 bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/sweep_c2_n$N.json 2> gpurun_out/sweep_c2_n$N.log; echo c2 rc=$?
fi
python -c "
import json; d=json.load(open('gpurun_out/sweep_c2_n$N.json')); print('c2', d['ms_per_step'], d['parity'], round(d['roofline']['frac'],4), d['e2e']['seconds'])"
bash scripts/gpu/gcfg.sh
