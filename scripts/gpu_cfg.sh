set -x
timeout 600 python -m pytest tests/test_gpu_local.py -q -x > gpurun_out/pytest_cfg.log 2>&1; echo pytest_rc=$?
for c in 0 1 2; do
  SPG_DENSE_CFG=$c timeout 600 python -m pytest tests/test_gpu_local.py -q -x -k "every_bin or merge_dense or rmat14" > gpurun_out/pytest_cfg$c.log 2>&1; echo cfg$c pytest_rc=$?
  SPG_DENSE_CFG=$c python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_cfg$c.json 2> gpurun_out/bench_cfg$c.err
  tail -1 gpurun_out/bench_cfg$c.err
done
python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"hash_rows" -c 2 -o gpurun_out/prof_hash \
    python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_hash.log 2>&1
echo ncu_rc=$?
