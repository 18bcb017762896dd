for e in 0 1; do
SPG_ESC1K=$e timeout 600 python -m pytest tests/test_gpu_local.py -q -m gpu -x > gpurun_out/pytest_esc$e.log 2>&1; echo "esc1k $e pytest_rc=$?"; tail -2 gpurun_out/pytest_esc$e.log
for w in "rmat --scale 18 --sr tropical_i32 --permute" "stencil --N 100 --sr arithmetic" "er --n-log2 20 --d 24 --sr arithmetic" "er --n-log2 16 --d 64 --sr maxtimes --value-mode 1"; do
  echo "== esc1k $e $w"
  SPG_ESC1K=$e timeout 300 python tools/local_probe.py $w --reps 3 2>/dev/null | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f bins %s' % (d['ms_total'], d['ms_numeric'], d['ms_compact'], d['rows_per_bin']))"
done
done
