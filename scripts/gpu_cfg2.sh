set -x
for c in 1 3; do
  SPG_DENSE_CFG=$c timeout 600 python -m pytest tests/test_gpu_local.py -q -x -k "every_bin or merge_dense or rmat14" > gpurun_out/pytest_cfg$c.log 2>&1; echo cfg$c pytest_rc=$?
  SPG_DENSE_CFG=$c python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
  tail -1 gpurun_out/bench_cfg$c.err; python -c "import json;d=json.load(open('gpurun_out/bench_cfg$c.json'));print('cfg$c', d['ms_per_step'])"
done
