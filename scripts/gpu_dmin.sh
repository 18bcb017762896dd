for dm in 4096 6144 8192; do
  echo "== dense_min $dm"
  SPG_DENSE_MIN=$dm timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 2 2>&1 | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f bins %s' % (d['ms_total'], d['ms_numeric'], d['ms_compact'], d['rows_per_bin']))"
done
