for cfg in 1 6; do
for fr in "0 1e12" "4096 16384" "16384 65536" "65536 262144" "262144 1e12"; do
  echo "== cfg $cfg F in ($fr]"
  SPG_DENSE_CFG=$cfg timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 2 --frange $fr 2>&1 | grep -v "^gen" | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f' % (d['ms_total'], d['ms_numeric'], d['ms_compact']))
    else: print('  ', l.strip())"
done
done
