timeout 900 python -m pytest tests/test_gpu_bitmap_rank.py tests/test_gpu_local.py -x -q -k "not headline" 2>&1 | tail -4
timeout 1500 python bench.py --config 3 --gpus 1 --summa --steps 2 --warmup 3 --e2e-steps 0 > gpurun_out/c3_n1b.json 2> gpurun_out/c3_n1b.log
echo rc=$?; tail -2 gpurun_out/c3_n1b.log; python -c "
import json; d=json.load(open('gpurun_out/c3_n1b.json')); print({k: d.get(k) for k in ('value','ms_per_step','parity','output')}, d['config']['nnz_C'], d['roofline']['frac'], d['config']['rank0_ledger']['batches'])"
