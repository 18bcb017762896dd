export PYTHONUNBUFFERED=1
timeout 1500 python bench.py --config 3 --gpus 1 --summa --steps 2 --warmup 3 --e2e-steps 0 > gpurun_out/c3_n1.json 2> gpurun_out/c3_n1.log
echo rc=$?; tail -5 gpurun_out/c3_n1.log; python -c "
import json; d=json.load(open('gpurun_out/c3_n1.json')); print({k: d.get(k) for k in ('value','ms_per_step','parity','output')}, d['config']['nnz_C'], d['config']['products'], d['roofline']['frac'], d['config']['rank0_ledger']['batches'])"
