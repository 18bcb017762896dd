set -x
N=$(nvidia-smi -L | wc -l)
export SPG_COMM_TIMEOUT_S=120 SPG_DEBUG_HANG=400
timeout 300 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/p1.json 2> gpurun_out/p1.err; echo p1 rc=$?
tail -1 gpurun_out/p1.err; cat gpurun_out/p1.json
timeout 450 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --steps 6 --warmup 3 --e2e-steps 0 > gpurun_out/p$N.json 2> gpurun_out/p$N.err; echo p$N rc=$?
cat gpurun_out/p$N.json
