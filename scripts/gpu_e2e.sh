set -x
timeout 900 python -m pytest tests -q -m gpu -x -k "not summa" > gpurun_out/pytest_e2e.log 2>&1; echo pytest_rc=$?
tail -2 gpurun_out/pytest_e2e.log
timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/e2e.json 2> gpurun_out/e2e.err; echo rc=$?
cat gpurun_out/e2e.json; tail -2 gpurun_out/e2e.err
