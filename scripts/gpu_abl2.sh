for v in default $(ls variants 2>/dev/null); do
  if [ "$v" = default ]; then unset SPG_LIB_PATH; else export SPG_LIB_PATH=$PWD/variants/$v/libspgemm_b200.so; fi
  for fr in "4096 1e12" "0 1e12"; do
  echo "== $v $fr"
  timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 2 --frange $fr 2>/dev/null | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f' % (d['ms_total'], d['ms_numeric'], d['ms_compact']))"
  done
done
