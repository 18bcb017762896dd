timeout 900 python -m pytest tests/test_gpu_local.py -x -q -m gpu > gpurun_out/ggred_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/ggred_tests.log
for g in 1 0; do
SPG_HASH_GRED=$g timeout 900 python bench.py --config 4 --summa --gpus 1 --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/c4_gred$g.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/c4_gred$g.json')); print('gred=$g', d['ms_per_step'], d['roofline'].get('frac'), d['config']['rank0_ledger']['ms'], d['config'].get('checksum_C'))"
done
