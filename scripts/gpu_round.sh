#!/bin/bash
# Round measurement set: default bench N=1/2/4, reference arm, launch list + ncu full of the dense kernel
mkdir -p gpurun_out/round
O=gpurun_out/round
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "n1 rc=$?"
timeout 900 $TR --nproc-per-node 2 --master-port 29541 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err; echo "n2 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29542 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err; echo "n4 rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/ref_n1.json 2> $O/ref_n1.err; echo "ref rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29543 bench.py --gpus 4 --config 4 --grid 1x4 --steps 3 --e2e-steps 0 > $O/c4_1x4.json 2> $O/c4_1x4.err; echo "c4 1x4 rc=$?"
export CUDA_VISIBLE_DEVICES=0
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_n1.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_panel -c 1 -o $O/dense_full python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
for f in bench_n1 bench_n2 bench_n4 ref_n1 c4_1x4; do echo "== $f"; cut -c1-400 $O/$f.json; done
