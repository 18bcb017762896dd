set -x
N=$(nvidia-smi -L | wc -l)
export SPG_COMM_TIMEOUT_S=120 SPG_DEBUG_HANG=400
timeout 450 python bench.py --steps 3 --warmup 3 --e2e-steps 1 > gpurun_out/n1.json 2> gpurun_out/n1.err; echo n1 rc=$?
cat gpurun_out/n1.json
timeout 450 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --steps 3 --warmup 3 > gpurun_out/n$N.json 2> gpurun_out/n$N.err; echo n$N rc=$?
cat gpurun_out/n$N.json
