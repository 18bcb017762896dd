mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "not summa" > gpurun_out/pytest_iter.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_iter.log
for w in "rmat --scale 18 --sr tropical_i32 --permute" "er --n-log2 16 --d 64 --sr maxtimes --value-mode 1" "er --n-log2 16 --d 64 --sr tropical_i32" "stencil --N 100 --sr arithmetic"; do
  echo "== $w"
  timeout 300 python tools/local_probe.py $w --reps 3 2>/dev/null | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f bins %s mode %s' % (d['ms_total'], d['ms_numeric'], d['ms_compact'], d['rows_per_bin'], d['output_mode']))"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_iter.csv python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_iter.csv | sort -rn | head -8
