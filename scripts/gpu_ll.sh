ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_now.csv python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > /dev/null 2>&1
python scripts/launches.py gpurun_out/launch_now.csv | sort -rn | head -12
