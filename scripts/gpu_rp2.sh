for mf in 0 16384 32768 65536; do
  echo "== rp_maxf $mf"
  SPG_RP_MAXF=$mf timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 3 2>/dev/null | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f bins %s' % (d['ms_total'], d['ms_numeric'], d['ms_compact'], d['rows_per_bin']))"
done
