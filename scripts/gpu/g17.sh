timeout 900 python -m pytest tests/test_gpu_summa.py -x -q -k "streamed" 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_local.py -x -q -k "row_batched" 2>&1 | tail -3
