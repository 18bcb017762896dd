timeout 900 python -m pytest tests/test_gpu_local.py tests/test_gpu_bitmap_rank.py tests/test_custom_semiring.py -x -q -k "not headline" 2>&1 | tail -4
timeout 600 python tools/local_probe.py stencil --N 252 --sr arithmetic --reps 3 2>&1 | grep -v "^gen" | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print({k: d[k] for k in ('ms_total','ms_numeric','ms_compact','rows_per_bin','output_mode')})
    else: print(l.strip()[:200])"
SPG_WARP_HASH=0 timeout 600 python tools/local_probe.py stencil --N 252 --sr arithmetic --reps 2 2>&1 | grep -o '"ms_total": [0-9.]*' | tail -1
timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 3 2>&1 | grep -o '"ms_total": [0-9.]*' | tail -1
