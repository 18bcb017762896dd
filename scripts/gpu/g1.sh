set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_bitmap_rank.py -x -q -k "not headline" 2>&1 | tail -15
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/b1.json 2> gpurun_out/b1.log; tail -5 gpurun_out/b1.log; cat gpurun_out/b1.json | head -c 1500
timeout 600 python -m pytest tests/test_gpu_bitmap_rank.py -x -q -k "headline" 2>&1 | tail -5
