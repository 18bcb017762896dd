# BASELINE configs 3-5 on one GPU (SUMMA 1x1; C streamed when larger than HBM), parity vs the oracle goldens
N=$(nvidia-smi -L | wc -l)
rm -f gpurun_out/configs_n$N.jsonl
for c in 3 4 5; do
  if [ "$N" = 1 ]; then
    timeout 1500 python bench.py --config $c --summa --gpus 1 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline >> gpurun_out/configs_n$N.jsonl 2>> gpurun_out/configs_n$N.log
  else
    timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2955$c bench.py --config $c --gpus $N --steps 2 --warmup 3 --e2e-steps 0 >> gpurun_out/configs_n$N.jsonl 2>> gpurun_out/configs_n$N.log
  fi
  echo c$c rc=$?
done
python -c "
import json
for l in open('gpurun_out/configs_n$N.jsonl'):
    d=json.loads(l); print(d['config']['workload'][:40], d['config'].get('grid'), d['ms_per_step'], d['parity'], round(d['roofline']['frac'],4), d.get('output'))"
