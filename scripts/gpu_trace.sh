mkdir -p gpurun_out
export SPG_HOST_TRACE=1
timeout 200 python tools/local_probe.py er --n-log2 20 --d 16 --sr boolean --reps 8 > gpurun_out/trace.txt 2>&1
timeout 200 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 8 >> gpurun_out/trace.txt 2>&1
cut -c1-220 gpurun_out/trace.txt
timeout 600 python -m pytest tests -q -m gpu -x -k "not summa" > gpurun_out/pytest_iter.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_iter.log
unset SPG_HOST_TRACE
python bench.py --steps 10 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_iter.json'));print(d['ms_per_step'],d['config'].get('steps_ms'))"; tail -1 gpurun_out/bench_iter.err
