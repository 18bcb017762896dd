timeout 600 python -m pytest tests/test_gpu_bitmap_rank.py -x -q -k "not headline" 2>&1 | grep -E "Error|error|passed|failed|assert" | head -12
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/b13.json 2> gpurun_out/b13.log; tail -1 gpurun_out/b13.log; head -c 300 gpurun_out/b13.json; echo
SPG_BR_WS=0 timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 3 2>&1 | grep -o '"ms_total": [0-9.]*' | tail -1
timeout 300 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 3 2>&1 | grep -o '"ms_total": [0-9.]*' | tail -1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/l13.csv python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > gpurun_out/l13.log 2>&1
