timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/b14.json 2> gpurun_out/b14.log; tail -3 gpurun_out/b14.log; python -c "
import json; d=json.load(open('gpurun_out/b14.json')); print({k: d[k] for k in ('value','ms_per_step','parity')}, d['config']['unpermuted'], d['roofline']['frac'], d['e2e'], d['cpu_baseline'])"
timeout 600 python -m pytest tests/test_gpu_local.py -x -q 2>&1 | tail -3
