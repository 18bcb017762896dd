for fr in "4096 16384" "16384 65536" "65536 262144" "262144 1e12" "4096 1e12"; do
  echo "== F in ($fr]"
  timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 3 --frange $fr 2>&1 | grep -v "^gen" | tail -2 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f bins %s' % (d['ms_total'], d['ms_numeric'], d['ms_compact'], d['rows_per_bin']))
    else: print('  ', l.strip())"
done
