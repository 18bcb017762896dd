timeout 1200 python -m pytest tests/test_gpu_summa.py -x -q -k "per_round or streamed or grids_on_one" 2>&1 | tail -4
