export VARIANTS="flat0"
bash scripts/gpu/ab.sh
bash scripts/gpu/ab.sh
bash scripts/gpu/ab.sh
timeout 600 python -m pytest tests/test_gpu_bitmap_rank.py tests/test_custom_semiring.py -x -q -m gpu 2>&1 | tail -2
