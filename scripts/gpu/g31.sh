N=$(nvidia-smi -L | wc -l)
if [ "$N" = 1 ]; then
timeout 1500 python bench.py --config 3 --gpus 1 --summa --steps 2 --warmup 3 --e2e-steps 0 > gpurun_out/c3_n1c.json 2> gpurun_out/c3_n1c.log
else
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --config 3 --gpus $N --steps 2 --warmup 3 --e2e-steps 0 > gpurun_out/c3_n$N.json 2> gpurun_out/c3_n$N.log
fi
echo rc=$?; python -c "
import json; d=json.load(open('gpurun_out/c3_n${N}$( [ $N = 1 ] && echo c).json')); print({k: d.get(k) for k in ('value','ms_per_step','parity','output','n_gpus')}, d['config']['grid'], d['roofline']['frac'], d['config']['rank0_ledger']['batches'])"
