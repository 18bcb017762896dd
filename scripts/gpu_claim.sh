mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_all.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_all.log
timeout 200 python tools/local_probe.py er --n-log2 16 --d 64 --sr maxtimes --value-mode 1 --reps 3 2>&1 | tail -1 | cut -c1-250
timeout 200 python tools/local_probe.py stencil --N 100 --sr arithmetic --reps 3 2>&1 | tail -1 | cut -c1-250
python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_iter.json'));print(d['ms_per_step'],d['config'].get('steps_ms'))"; tail -1 gpurun_out/bench_iter.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/c4_n1.json 2> gpurun_out/c4_n1.err; echo "c4 n1 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/c4_n1.json'));c=d['config'];print(d['value'],d['ms_per_step'],c['matches_expected'],c['per_rank_ms'])"
