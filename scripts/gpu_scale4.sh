set -x
export SPG_COMM_TIMEOUT_S=120 SPG_DEBUG_HANG=400
timeout 900 python -m pytest tests/test_gpu_summa.py -q -x > gpurun_out/pytest_summa4.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_summa4.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/sc1.json 2> gpurun_out/sc1.err; echo rc1=$?
for N in 2 4; do
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2954$N \
  bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/sc$N.json 2> gpurun_out/sc$N.err; echo rc$N=$?
done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29549 \
  bench.py --gpus 4 --grid 1x4 --steps 5 --warmup 3 > gpurun_out/sc4b.json 2> gpurun_out/sc4b.err; echo rc4b=$?
