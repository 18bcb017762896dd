for cfg in 7 8; do
SPG_DENSE_CFG=$cfg timeout 600 python -m pytest tests/test_gpu_local.py -q -m gpu -x > gpurun_out/pytest_ws$cfg.log 2>&1; echo "cfg $cfg pytest_rc=$?"; tail -2 gpurun_out/pytest_ws$cfg.log
done
for cfg in 1 7 8; do
for fr in "0 1e12" "4096 1e12"; do
  echo "== cfg $cfg $fr"
  SPG_DENSE_CFG=$cfg timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 2 --frange $fr 2>/dev/null | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f nnz %d' % (d['ms_total'], d['ms_numeric'], d['ms_compact'], d['nnz_out']))"
done
done
