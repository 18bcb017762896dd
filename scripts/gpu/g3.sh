set -x
timeout 900 python -m pytest tests/test_gpu_bitmap_rank.py tests/test_gpu_local.py -x -q 2>&1 | tail -8
timeout 300 python bench.py --steps 5 --warmup 3 > gpurun_out/b3.json 2> gpurun_out/b3.log; tail -3 gpurun_out/b3.log; head -c 600 gpurun_out/b3.json
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/l3.csv python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > gpurun_out/l3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:br_numeric -c 1 -o gpurun_out/br_num3 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > gpurun_out/n3.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:br_symbolic -c 1 -o gpurun_out/br_sym3 python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > gpurun_out/s3.log 2>&1
