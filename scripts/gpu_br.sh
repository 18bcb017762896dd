timeout 600 python -m pytest tests/test_gpu_local.py -q -m gpu -x > gpurun_out/pytest_br.log 2>&1; echo "pytest_rc=$?"; tail -2 gpurun_out/pytest_br.log
for b in 0 1; do
for w in "rmat --scale 18 --sr tropical_i32 --permute" "rmat --scale 18 --sr tropical_i32 --permute --frange 512 16384" "er --n-log2 16 --d 64 --sr tropical_i32" "rmat --scale 16 --sr boolean --permute"; do
  echo "== bitrank $b $w"
  SPG_BITRANK=$b timeout 300 python tools/local_probe.py $w --reps 3 2>/dev/null | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f bins %s nnz %d' % (d['ms_total'], d['ms_numeric'], d['ms_compact'], d['rows_per_bin'], d['nnz_out']))"
done
done
