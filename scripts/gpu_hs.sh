timeout 900 python -m pytest tests/test_gpu_local.py -q -m gpu -x > gpurun_out/pytest_hs.log 2>&1; echo "pytest_rc=$?"; tail -1 gpurun_out/pytest_hs.log
for w in "rmat --scale 18 --sr tropical_i32 --permute" "stencil --N 100 --sr arithmetic" "er --n-log2 16 --d 64 --sr maxtimes --value-mode 1" "er --n-log2 20 --d 16 --sr tropical_i32"; do
  echo "== $w"
  timeout 300 python tools/local_probe.py $w --reps 3 2>/dev/null | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f' % (d['ms_total'], d['ms_numeric'], d['ms_compact']))"
done
