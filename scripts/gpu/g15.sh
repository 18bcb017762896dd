timeout 900 python -m pytest tests/test_gpu_layout.py tests/test_gpu_summa.py -x -q 2>&1 | tail -15
