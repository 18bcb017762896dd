for fr in "0 1e12" "4096 1e12"; do
  echo "== F in ($fr]"
  timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 3 --frange $fr 2>&1 | grep -v "^gen" | tail -2 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f bins %s mode %s' % (d['ms_total'], d['ms_numeric'], d['ms_compact'], d['rows_per_bin'], d['output_mode']))
    else: print('  ', l.strip())"
done
echo "== plain"
timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 3 2>&1 | tail -1 | cut -c1-300
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_sub.csv python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 --frange 4096 1e12 > /dev/null 2>&1
python scripts/launches.py gpurun_out/launch_sub.csv | sort -rn | head -4
