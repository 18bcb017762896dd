timeout 900 python bench.py --config 4 --summa --gpus 1 --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/c4_sorted.json 2> gpurun_out/c4_sorted.log; echo rc=$?
python -c "
import json; d=json.load(open('gpurun_out/c4_sorted.json')); print(d['ms_per_step'], d['value'], d['roofline'].get('frac'), d['config']['rank0_ledger']['ms'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:hash_rows_kernel -c 2 --csv --log-file gpurun_out/c4_252_sorted.csv python bench.py --config 4 --summa --gpus 1 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
cat gpurun_out/c4_252_sorted.csv | grep -v "^==" | cut -c1-400 | tail -6
