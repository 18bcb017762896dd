#!/bin/bash
mkdir -p gpurun_out/round
O=gpurun_out/round
timeout 900 python -m pytest tests -q -m gpu -x > $O/pytest_all.log 2>&1; echo pytest_rc=$?; tail -2 $O/pytest_all.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/traffic_n1.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29543 bench.py --gpus 4 --config 4 --steps 3 --e2e-steps 0 > $O/c4_n4.json 2> $O/c4_n4.err; echo "c4 rc=$?"
cut -c1-300 $O/c4_n4.json
