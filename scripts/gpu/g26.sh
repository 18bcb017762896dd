timeout 600 python -m pytest tests/test_gpu_bitmap_rank.py -x -q -k "not headline" 2>&1 | tail -2
bash scripts/gpu/prof.sh
timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 4 2>&1 | grep -o '"ms_total": [0-9.]*' | tail -2
