timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > gpurun_out/r02_launches.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:br_numeric -c 1 -o gpurun_out/r02_br_numeric python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:br_symbolic -c 1 -o gpurun_out/r02_br_symbolic python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > /dev/null 2>&1
ls -la gpurun_out | grep r02
