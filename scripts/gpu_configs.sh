#!/bin/bash
# BASELINE configs 3, 4, 5 at full size on a 4-GPU box; config 4 also at 1 and 2 GPUs
mkdir -p gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
B="--steps 3 --warmup 3 --e2e-steps 0"
timeout 900 python bench.py --config 4 $B > gpurun_out/c4_n1.json 2> gpurun_out/c4_n1.err; echo "c4 n1 rc=$?"
timeout 900 $TR --nproc-per-node 2 --master-port 29531 bench.py --gpus 2 --config 4 $B > gpurun_out/c4_n2.json 2> gpurun_out/c4_n2.err; echo "c4 n2 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29532 bench.py --gpus 4 --config 4 $B > gpurun_out/c4_n4.json 2> gpurun_out/c4_n4.err; echo "c4 n4 rc=$?"
timeout 1200 $TR --nproc-per-node 4 --master-port 29533 bench.py --gpus 4 --config 5 $B > gpurun_out/c5_n4.json 2> gpurun_out/c5_n4.err; echo "c5 n4 rc=$?"
timeout 1500 $TR --nproc-per-node 4 --master-port 29534 bench.py --gpus 4 --config 3 $B > gpurun_out/c3_n4.json 2> gpurun_out/c3_n4.err; echo "c3 n4 rc=$?"
for f in c4_n1 c4_n2 c4_n4 c5_n4 c3_n4; do echo "== $f"; python -c "
import json;d=json.load(open('gpurun_out/$f.json'));c=d['config'];print(d['value'],d['ms_per_step'],c['products'],c['nnz_C'],c.get('matches_expected'),c['steps_ms_max_over_ranks']); print(c['per_rank_ms'])" 2>&1 | tail -2; grep -v "^\[rank\|NCCL" gpurun_out/$f.err | tail -2; done
