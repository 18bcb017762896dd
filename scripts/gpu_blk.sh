for b in "1 1 0 0" "1 2 0 0" "2 2 0 0" "2 2 1 1"; do
  echo "== block $b"
  timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 3 --block $b 2>&1 | grep -v "^gen" | tail -2 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f F %.3g bins %s' % (d['ms_total'], d['ms_numeric'], d['ms_compact'], d['products'], d['rows_per_bin']))
    else: print('  ', l.strip())"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_blk.csv python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 --block 2 2 0 0 > /dev/null 2>&1
python scripts/launches.py gpurun_out/launch_blk.csv | sort -rn | head -10
