# A/B of library variants on the config-2 local multiply: python tools/local_probe.py per variant
for v in base $VARIANTS; do
  if [ "$v" = base ]; then export -n SPG_LIB_PATH; unset SPG_LIB_PATH; else export SPG_LIB_PATH=variants/$v/libspgemm_b200.so; fi
  timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 6 2>/dev/null | python -c "
import sys, json
r=[json.loads(l) for l in sys.stdin if l.startswith('{')]
t=sorted(x['ms_total'] for x in r[1:]); print('$v', 'ms_total median %.2f min %.2f' % (t[len(t)//2], t[0]), 'numeric', round(sorted(x['ms_numeric'] for x in r[1:])[len(r)//2-1],2))"
done
