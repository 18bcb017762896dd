# A/B of library variants x dense configs on the config-2 local multiply (permuted R-MAT s18 tropical)
mkdir -p gpurun_out
for v in default $(ls variants 2>/dev/null); do
  if [ "$v" = default ]; then unset SPG_LIB_PATH; else export SPG_LIB_PATH=$PWD/variants/$v/libspgemm_b200.so; fi
  for cfg in ${CFGS:-1}; do
  echo "== $v cfg $cfg"
  SPG_DENSE_CFG=$cfg timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 4 2>/dev/null | tail -2 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f analyse %.2f' % (d['ms_total'], d['ms_numeric'], d['ms_compact'], d['ms_analyse']))"
  done
done
unset SPG_LIB_PATH
