timeout 600 python -m pytest tests/test_gpu_bitmap_rank.py -x -q 2>&1 | tail -4
timeout 900 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_bitmap_rank.py -x -q -k "same_as_bins" 2>&1 | grep -v "^    " | head -40
