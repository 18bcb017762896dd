timeout 900 python -m pytest tests/test_gpu_local.py -x -q -m gpu > gpurun_out/gwide.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gwide.log
timeout 1800 python bench.py --config 5 --summa --gpus 1 --steps 1 --warmup 3 --e2e-steps 0 > gpurun_out/c5_n1.json 2> gpurun_out/c5_n1.log; echo c5 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/c5_n1.json')); print({k: d.get(k) for k in ('value','unit','ms_per_step','parity','output')}, d['roofline'].get('frac'), d['config'].get('rank0_ledger',{}).get('batches'))"
grep -v "^\[rank0\]:   " gpurun_out/c5_n1.log | tail -5
# config-4 hash kernel: one full ncu capture (stencil N=96, 1x1 SUMMA path)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hash_rows_kernel -c 1 -o gpurun_out/c4_hash python bench.py --config 4 --stencil-n 96 --summa --gpus 1 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/c4_hash_ncu.log 2>&1; echo ncu rc=$?
