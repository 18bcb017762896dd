#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/local_probe.py er --n-log2 16 --d 64 --sr maxtimes --value-mode 1 > gpurun_out/probe_er.txt 2>&1; echo rc=$?
timeout 120 python tools/local_probe.py er --n-log2 16 --d 64 --sr tropical_i32 --reps 3 >> gpurun_out/probe_er.txt 2>&1
timeout 120 python tools/local_probe.py er --n-log2 16 --d 64 --sr arithmetic --reps 3 >> gpurun_out/probe_er.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:hash_rows -c 1 -o gpurun_out/er_hash python tools/local_probe.py er --n-log2 16 --d 64 --sr maxtimes --value-mode 1 --reps 1 > gpurun_out/ncu_er.log 2>&1; echo ncu rc=$?
timeout 120 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/er_launches.csv python tools/local_probe.py er --n-log2 16 --d 64 --sr maxtimes --value-mode 1 --reps 1 > /dev/null 2>&1
cat gpurun_out/probe_er.txt
