timeout 900 python -m pytest tests/test_gpu_local.py -x -q -m gpu -k "download or wide or sorted" > gpurun_out/gdl.log 2>&1; echo rc=$?; tail -3 gpurun_out/gdl.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-unpermuted > gpurun_out/bench_e2e1.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/bench_e2e1.json')); print(d['ms_per_step'], d['e2e'], d['parity'])"
