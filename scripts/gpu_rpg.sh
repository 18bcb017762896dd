timeout 900 python -m pytest tests/test_gpu_local.py -q -m gpu -x > gpurun_out/pytest_rpg.log 2>&1; echo "pytest_rc=$?"; tail -1 gpurun_out/pytest_rpg.log
SPG_RP_GEOM=2 timeout 900 python -m pytest tests/test_gpu_local.py -q -m gpu -x -k "bitrank or rank_panel or every_bin" > gpurun_out/pytest_rpg2.log 2>&1; echo "pytest2_rc=$?"; tail -1 gpurun_out/pytest_rpg2.log
for g in 1 2; do
for mf in 16384 32768; do
  echo "== geom $g maxf $mf"
  SPG_RP_GEOM=$g SPG_RP_MAXF=$mf timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 3 2>/dev/null | tail -1 | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  total %.2f numeric %.2f compact %.2f bins %s' % (d['ms_total'], d['ms_numeric'], d['ms_compact'], d['rows_per_bin']))"
done
done
