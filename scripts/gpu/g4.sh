timeout 900 python -m pytest tests/test_gpu_bitmap_rank.py -x -q -k "not headline" 2>&1 | tail -4
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/b4.json 2> gpurun_out/b4.log; tail -2 gpurun_out/b4.log; head -c 400 gpurun_out/b4.json; echo
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/l4.csv python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > gpurun_out/l4.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:br_numeric -c 1 -o gpurun_out/br_num4 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > gpurun_out/n4.log 2>&1
