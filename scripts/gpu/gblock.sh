for b in "1 1 0 0" "1 2 0 0" "2 2 0 0" "2 2 1 1"; do
timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --block $b --reps 6 2>/dev/null | python -c "
import sys, json
r=[json.loads(l) for l in sys.stdin if l.startswith('{')]
t=sorted(x['ms_total'] for x in r[1:]); x=r[-1]
print('$b', 'ms_total %.2f' % t[len(t)//2], 'products', x['products'], 'sym %.2f fold %.2f' % (x['ms_symbolic'], x['ms_fold']), 'mode', x['output_mode'], 'bins', x['rows_per_bin'])"
done
