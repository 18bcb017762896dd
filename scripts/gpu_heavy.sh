timeout 600 python -m pytest tests/test_gpu_local.py -q -m gpu -x > gpurun_out/pytest_h.log 2>&1; echo "pytest_rc=$?"; tail -1 gpurun_out/pytest_h.log
for h in 0 1; do
for w in "rmat --scale 18 --sr tropical_i32 --permute" "rmat --scale 18 --sr tropical_i32" "rmat --scale 16 --sr boolean --permute"; do
  echo "== heavy $h $w"
  SPG_DENSE_HEAVY=$h timeout 300 python tools/local_probe.py $w --reps 3 2>/dev/null | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f mode %d' % (d['ms_total'], d['ms_numeric'], d['ms_compact'], d['output_mode']))"
done
done
