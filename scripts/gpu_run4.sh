set -x
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu4.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/pytest_gpu4.log
python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench_rc=$?
cat gpurun_out/bench4.json; tail -3 gpurun_out/bench4.err
python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches4.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu4.log 2>&1
echo ncu_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"dense_panel|esc_block" -c 4 -o gpurun_out/prof4 \
    python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu4full.log 2>&1
echo ncufull_rc=$?
