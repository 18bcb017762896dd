mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_panel -c 1 -o gpurun_out/dense_r01b python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > gpurun_out/ncu_dense.log 2>&1; echo ncu_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hash_rows -c 2 -o gpurun_out/hash_r01b python tools/local_probe.py rmat --scale 18 --sr tropical_i32 --permute --reps 1 > gpurun_out/ncu_hash.log 2>&1; echo ncu_rc=$?
