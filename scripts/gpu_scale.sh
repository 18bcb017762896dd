set -x
export SPG_COMM_TIMEOUT_S=120 SPG_DEBUG_HANG=400
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sc1.json 2> gpurun_out/sc1.err; echo rc1=$?
for N in 2 4 8; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N \
  bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/sc$N.json 2> gpurun_out/sc$N.err; echo rc$N=$?
done
