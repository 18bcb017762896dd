timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c3_batch.csv python tools/local_probe.py rmat --scale 22 --sr boolean --frange 300000 1000000 --reps 1 > gpurun_out/c3_batch.log 2>&1
tail -3 gpurun_out/c3_batch.log
