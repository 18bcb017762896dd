timeout 600 python -m pytest tests/test_gpu_bitmap_rank.py tests/test_gpu_local.py -x -q -k "not headline" 2>&1 | tail -4
