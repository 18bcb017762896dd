timeout 900 python -m pytest tests/test_gpu_bitmap_rank.py -x -q -m gpu > gpurun_out/gc3c_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gc3c_tests.log
timeout 1500 python bench.py --config 3 --summa --gpus 1 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/c3_c.json 2> gpurun_out/c3_c.log; echo c3 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/c3_c.json')); print(d['ms_per_step'], d['parity'], d['roofline']['frac'])"
