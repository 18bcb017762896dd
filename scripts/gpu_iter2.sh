# local parity + ER/R-MAT probes + bench + launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "not summa" > gpurun_out/pytest_iter.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_iter.log
timeout 120 python tools/local_probe.py er --n-log2 16 --d 64 --sr maxtimes --value-mode 1 --reps 3 > gpurun_out/probe_er.txt 2>&1
timeout 120 python tools/local_probe.py er --n-log2 16 --d 64 --sr tropical_i32 --reps 3 >> gpurun_out/probe_er.txt 2>&1

cat gpurun_out/probe_er.txt | cut -c1-250
python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo bench_rc=$?
cat gpurun_out/bench_iter.json; tail -2 gpurun_out/bench_iter.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_iter.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_iter.log 2>&1
echo ncu_rc=$?
