export VARIANTS="skip0"
bash scripts/gpu/ab.sh
bash scripts/gpu/ab.sh
for v in base skip0; do
  if [ "$v" = base ]; then unset SPG_LIB_PATH; else export SPG_LIB_PATH=variants/$v/libspgemm_b200.so; fi
  timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --reps 6 2>/dev/null | python -c "
import sys, json
r=[json.loads(l) for l in sys.stdin if l.startswith('{')]
t=sorted(x['ms_total'] for x in r[1:]); print('unpermuted $v', 'ms_total median %.2f' % t[len(t)//2])"
done
unset SPG_LIB_PATH
timeout 600 python -m pytest tests/test_gpu_bitmap_rank.py tests/test_custom_semiring.py -x -q -m gpu 2>&1 | tail -2
