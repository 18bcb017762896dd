mkdir -p gpurun_out
export SPG_HOST_TRACE=20
python bench.py --steps 3 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo bench_rc=$?
python -c "import json;d=json.load(open('gpurun_out/bench_iter.json'));print(d['ms_per_step'], d['e2e'])"; grep "spg-host" gpurun_out/bench_iter.err | tail -40
