set -x
timeout 600 python -m pytest tests/test_gpu_bitmap_rank.py -x -q -k "not headline" 2>&1 | tail -5
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/l2.csv python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > gpurun_out/l2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:br_numeric -c 1 -o gpurun_out/br_num python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > gpurun_out/n2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:br_symbolic -c 1 -o gpurun_out/br_sym python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > gpurun_out/s2.log 2>&1
ls -la gpurun_out
