#!/bin/bash
# BASELINE configs 3-5 at small sizes (closed forms / reference checks) + config 4 full size on 1 GPU
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --e2e-steps 0"
timeout 300 $B --config 4 --stencil-n 40 > gpurun_out/c4_small.json 2> gpurun_out/c4_small.err; echo "c4 small rc=$?"
timeout 300 $B --config 5 --er-log2 16 > gpurun_out/c5_small.json 2> gpurun_out/c5_small.err; echo "c5 small rc=$?"
timeout 300 $B --config 3 --scale 16 > gpurun_out/c3_small.json 2> gpurun_out/c3_small.err; echo "c3 small rc=$?"
timeout 900 $B --config 4 > gpurun_out/c4_n1.json 2> gpurun_out/c4_n1.err; echo "c4 full rc=$?"
tail -3 gpurun_out/*.err
