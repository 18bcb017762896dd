set -x
N=$(nvidia-smi -L | wc -l)
python bench.py --summa --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/summa1.json 2> gpurun_out/summa1.err; echo rc=$?
tail -3 gpurun_out/summa1.err; cat gpurun_out/summa1.json
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --steps 3 --warmup 3 > gpurun_out/summa$N.json 2> gpurun_out/summa$N.err; echo rc=$?
tail -5 gpurun_out/summa$N.err; cat gpurun_out/summa$N.json
timeout 900 python -m pytest tests/test_gpu_summa.py -q -x > gpurun_out/pytest_summa.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_summa.log
