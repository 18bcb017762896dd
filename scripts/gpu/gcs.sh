timeout 1200 python -m pytest tests/test_gpu_local.py tests/test_gpu_bitmap_rank.py tests/test_gpu_layout.py -x -q -m gpu > gpurun_out/gcs_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gcs_tests.log
timeout 1500 python bench.py --config 3 --summa --gpus 1 --steps 2 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/c3_cs.json 2> gpurun_out/c3_cs.log; echo c3 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/c3_cs.json')); print('c3', d['ms_per_step'], d['parity'], d['roofline']['frac'])"
timeout 1500 python bench.py --config 5 --summa --gpus 1 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/c5_cs.json 2> gpurun_out/c5_cs.log; echo c5 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/c5_cs.json')); print('c5', d['ms_per_step'], d['parity'], d['roofline']['frac'], d['config']['checksum_C'])"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-unpermuted > gpurun_out/c2_cs.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/c2_cs.json')); print('c2', d['ms_per_step'], d['parity'], d['roofline']['frac'])"
