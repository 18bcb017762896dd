set -x
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu3.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu3.log
python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo bench_rc=$?
cat gpurun_out/bench3.json; tail -3 gpurun_out/bench3.err
python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches3.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1
echo ncu_rc=$?
