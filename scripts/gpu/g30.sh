timeout 900 python -m pytest tests/test_gpu_bitmap_rank.py -x -q -k "pattern or rank_windows or same_as" 2>&1 | tail -2
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c3_batch2.csv python tools/local_probe.py rmat --scale 22 --sr boolean --frange 300000 1000000 --reps 1 > gpurun_out/c3_batch2.log 2>&1
grep -h "br_pattern" gpurun_out/c3_batch2.csv | awk -F'","' '{print $5, $NF}' | cut -c1-150
