timeout 600 python -m pytest tests/test_gpu_local.py -q -m gpu -x > gpurun_out/pytest_rp.log 2>&1; echo "pytest_rc=$?"; tail -1 gpurun_out/pytest_rp.log
for rp in 0 1; do
for w in "rmat --scale 18 --sr tropical_i32 --permute" "rmat --scale 18 --sr tropical_i32" "rmat --scale 16 --sr boolean --permute" "rmat --scale 18 --sr minplus --permute"; do
  echo "== rankpanel $rp $w"
  SPG_RANKPANEL=$rp timeout 300 python tools/local_probe.py $w --reps 3 2>/dev/null | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f bins %s nnz %d' % (d['ms_total'], d['ms_numeric'], d['ms_compact'], d['rows_per_bin'], d['nnz_out']))"
done
done
