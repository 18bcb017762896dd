timeout 900 python -m pytest tests/test_gpu_local.py tests/test_gpu_bitmap_rank.py -x -q -m gpu > gpurun_out/gdl2.log 2>&1; echo rc=$?; tail -2 gpurun_out/gdl2.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.log; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_default.json')); print(d['ms_per_step'], d['parity'], round(d['roofline']['frac'],4), d['e2e'])"
