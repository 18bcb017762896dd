#!/bin/bash
# final bench lines + launch/traffic list (4-GPU box)
mkdir -p gpurun_out/final
O=gpurun_out/final
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -q -m gpu > $O/pytest_all.log 2>&1; echo pytest_rc=$?; tail -1 $O/pytest_all.log
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "n1 rc=$?"
timeout 900 $TR --nproc-per-node 2 --master-port 29741 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err; echo "n2 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29742 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err; echo "n4 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref_n1.json 2> $O/ref_n1.err; echo "ref rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29743 bench.py --impl reference --gpus 4 --steps 1 --warmup 1 > $O/ref_n4.json 2> $O/ref_n4.err; echo "ref4 rc=$?"
export CUDA_VISIBLE_DEVICES=0
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/traffic_n1.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
for f in bench_n1 bench_n2 bench_n4 ref_n1 ref_n4; do echo "== $f"; python -c "
import json;d=json.load(open('$O/$f.json'));c=d['config'];print(d['value'],d['ms_per_step'],d.get('e2e'),c.get('steps_ms') or c.get('steps_ms_max_over_ranks'))" 2>&1 | tail -1; done
