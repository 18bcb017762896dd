export SPG_HOST_TRACE=20
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --config 5 --gpus 2 --steps 2 --warmup 3 --e2e-steps 0 > gpurun_out/c5_n2.json 2> gpurun_out/c5dbg2_n2.log; echo n2 rc=$?
grep "summa batch\|cudaMalloc\|release" gpurun_out/c5dbg2_n2.log | tail -40
python -c "
import json; d=json.load(open('gpurun_out/c5_n2.json')); c=d['config']; print(d['ms_per_step'], d['parity'], c['steps_ms_max_over_ranks'])"
unset SPG_HOST_TRACE
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-unpermuted > gpurun_out/c2_sc.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/c2_sc.json')); print('c2', d['ms_per_step'], d['parity'], d['e2e']['seconds'])"
