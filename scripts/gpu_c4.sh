mkdir -p gpurun_out
export SPG_HOST_TRACE=5
timeout 900 python bench.py --config 4 --steps 4 --warmup 3 --e2e-steps 0 > gpurun_out/c4_n1.json 2> gpurun_out/c4_n1.err; echo "c4 n1 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/c4_n1.json'));c=d['config'];print(d['value'],d['ms_per_step'],c['matches_expected'],c['steps_ms_max_over_ranks'],c['per_rank_ms'])"
grep "spg-host" gpurun_out/c4_n1.err | tail -30
unset SPG_HOST_TRACE
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_all.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_all.log
python bench.py --steps 10 --warmup 3 --e2e-steps 2 > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_iter.json'));print(d['ms_per_step'],d['config'].get('steps_ms'), d['e2e'])"; tail -1 gpurun_out/bench_iter.err
