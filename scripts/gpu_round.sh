#!/bin/bash
mkdir -p gpurun_out/round
O=gpurun_out/round
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 python -m pytest tests -q -m gpu -x > $O/pytest_all.log 2>&1; echo pytest_rc=$?; tail -1 $O/pytest_all.log
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "n1 rc=$?"
timeout 900 $TR --nproc-per-node 2 --master-port 29541 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err; echo "n2 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29542 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err; echo "n4 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref_n1.json 2> $O/ref_n1.err; echo "ref rc=$?"
B="--steps 3 --warmup 3 --e2e-steps 0"
timeout 900 $TR --nproc-per-node 4 --master-port 29543 bench.py --gpus 4 --config 4 $B > $O/c4_n4.json 2> $O/c4_n4.err; echo "c4 rc=$?"
timeout 1200 $TR --nproc-per-node 4 --master-port 29544 bench.py --gpus 4 --config 5 $B > $O/c5_n4.json 2> $O/c5_n4.err; echo "c5 rc=$?"
timeout 1500 $TR --nproc-per-node 4 --master-port 29545 bench.py --gpus 4 --config 3 $B > $O/c3_n4.json 2> $O/c3_n4.err; echo "c3 rc=$?"
timeout 900 python bench.py --config 4 $B > $O/c4_n1.json 2> $O/c4_n1.err; echo "c4n1 rc=$?"
export CUDA_VISIBLE_DEVICES=0
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/traffic_n1.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/ncu_traffic.log 2>&1; echo "ncu traffic rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_panel_kernel -c 2 -o $O/dense_full python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bitrank -c 1 -o $O/bitrank_full python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > $O/ncu_full2.log 2>&1; echo "ncu full2 rc=$?"
for f in bench_n1 bench_n2 bench_n4 ref_n1 c4_n4 c5_n4 c3_n4 c4_n1; do echo "== $f"; python -c "
import json;d=json.load(open('$O/$f.json'));c=d['config'];print(d['value'],d['ms_per_step'],c.get('steps_ms') or c.get('steps_ms_max_over_ranks'),c.get('matches_expected'))" 2>&1 | tail -1; done
