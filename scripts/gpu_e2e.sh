timeout 900 python -m pytest tests -q -m gpu -x -k "not summa" > gpurun_out/pytest_e2e.log 2>&1; echo "pytest_rc=$?"; tail -1 gpurun_out/pytest_e2e.log
python bench.py --steps 5 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_e2e.json'));print(d['ms_per_step'], d['e2e'])"
