for cfg in 1 0 2; do
for fr in "8192 65536" "65536 262144" "262144 1e12"; do
  echo "== cfg $cfg F in ($fr]"
  SPG_DENSE_CFG=$cfg timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 2 --frange $fr 2>&1 | grep -v "^gen\|^rows" | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f' % (d['ms_total'], d['ms_numeric'], d['ms_compact']))"
done
done
