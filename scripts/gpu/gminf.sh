for mf in 2048 1024 512; do
for b in "1 1 0 0" "1 2 0 0" "2 2 0 0"; do
SPG_BR_MINF=$mf timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --block $b --reps 6 2>/dev/null | python -c "
import sys, json
r=[json.loads(l) for l in sys.stdin if l.startswith('{')]
t=sorted(x['ms_total'] for x in r[1:]); x=r[-1]
print('minf $mf block $b', 'ms_total %.2f' % t[len(t)//2], 'sym %.2f fold %.2f' % (x['ms_symbolic'], x['ms_fold']), 'bitmap rows', x['rows_per_bin'][10])"
done; done
