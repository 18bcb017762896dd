for p in "--permute" ""; do
timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 $p --reps 5 2>/dev/null | python -c "
import sys, json
r=[json.loads(l) for l in sys.stdin if l.startswith('{')]
t=sorted(x['ms_total'] for x in r[1:]); x=r[-1]
print('perm=$p', 'ms_total %.2f' % t[len(t)//2], 'sym %.2f fold %.2f items %d bitmap_bytes %.2f GB' % (x['ms_symbolic'], x['ms_fold'], x['fold_items'], x['bitmap_bytes']/1e9), 'bins', x['rows_per_bin'])"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_unperm.csv python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --reps 1 > /dev/null 2>&1; echo ncu rc=$?
