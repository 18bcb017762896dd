timeout 600 python -m pytest tests/test_gpu_local.py -q -m gpu -x > gpurun_out/pytest_br.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_br.log
for v in off default; do
  if [ "$v" = default ] || [ "$v" = off ]; then unset SPG_LIB_PATH; else export SPG_LIB_PATH=$PWD/variants/$v/libspgemm_b200.so; fi
  if [ "$v" = off ]; then export SPG_BITRANK=0; else unset SPG_BITRANK; fi
for w in "rmat --scale 18 --sr tropical_i32 --permute" "er --n-log2 16 --d 64 --sr maxtimes --value-mode 1" "stencil --N 100 --sr minplus" "rmat --scale 16 --sr boolean --permute"; do
  echo "== $v $w"
  timeout 300 python tools/local_probe.py $w --reps 3 2>/dev/null | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f bins %s' % (d['ms_total'], d['ms_numeric'], d['ms_compact'], d['rows_per_bin']))"
done
done
