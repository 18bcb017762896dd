# config 4 at 1x1: optimistic 512-slot hash (default) vs the 2K table (SPG_HASH_OPT=0)
timeout 900 python bench.py --config 4 --summa --gpus 1 --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/c4_opt.json 2> gpurun_out/c4_opt.log; echo opt rc=$?
SPG_HASH_OPT=0 timeout 900 python bench.py --config 4 --summa --gpus 1 --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/c4_base.json 2> gpurun_out/c4_base.log; echo base rc=$?
for f in c4_opt c4_base; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', d['ms_per_step'], d['value'], d['roofline'].get('frac'), d.get('parity'))"; done
timeout 900 python -m pytest tests/test_gpu_local.py tests/test_gpu_bitmap_rank.py -x -q -m gpu > gpurun_out/gc4_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/gc4_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:hash_rows_kernel -c 20 --csv --log-file gpurun_out/c4_opt_launches.csv python bench.py --config 4 --stencil-n 128 --summa --gpus 1 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2>&1; echo ncu rc=$?
