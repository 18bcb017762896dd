# configs 4 and 5 on one GPU (SUMMA 1x1 path; C streamed when it exceeds HBM) + launch list of config 4 at N=128
timeout 900 python bench.py --config 4 --summa --gpus 1 --steps 2 --warmup 3 --e2e-steps 0 > gpurun_out/c4_n1.json 2> gpurun_out/c4_n1.log; echo c4 rc=$?
timeout 1800 python bench.py --config 5 --summa --gpus 1 --steps 1 --warmup 3 --e2e-steps 0 > gpurun_out/c5_n1.json 2> gpurun_out/c5_n1.log; echo c5 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/c4_launches.csv python bench.py --config 4 --stencil-n 128 --summa --gpus 1 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/c4_ncu.log 2>&1; echo ncu4 rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/c5_launches.csv python bench.py --config 5 --er-log2 19 --summa --gpus 1 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/c5_ncu.log 2>&1; echo ncu5 rc=$?
for f in c4_n1 c5_n1; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', {k: d.get(k) for k in ('value','unit','ms_per_step','parity','output')}, d['roofline'].get('frac'), d['config'].get('rank0_ledger',{}).get('batches'))"; done
