# quick iteration: GPU parity (local kernels) + bench + launch list
set -x
timeout 900 python -m pytest tests -q -m gpu -x -k "not summa" > gpurun_out/pytest_iter.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_iter.log
python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_iter.json 2> gpurun_out/bench_iter.err; echo bench_rc=$?
cat gpurun_out/bench_iter.json; tail -2 gpurun_out/bench_iter.err
python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_iter.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_iter.log 2>&1
echo ncu_rc=$?
if [ -n "$SPG_NCU_FULL" ]; then
ncu --set full --clock-control none --import-source on -k regex:"$SPG_NCU_FULL" -c 1 -o gpurun_out/prof_iter \
    python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full_iter.log 2>&1
echo ncufull_rc=$?
fi
