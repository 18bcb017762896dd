set -x
N=$(nvidia-smi -L | wc -l)
export SPG_COMM_TIMEOUT_S=120 SPG_DEBUG_HANG=400
timeout 900 python -m pytest tests/test_gpu_summa.py tests/test_cpp_facade.py -q -x > gpurun_out/pytest_summa.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/pytest_summa.log
timeout 300 python bench.py --summa --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/s1.json 2> gpurun_out/s1.err; echo s1 rc=$?
python -c "import json;d=json.load(open('gpurun_out/s1.json'));print(d['value'],d['ms_per_step'],d['config']['rank0_ledger'])"
timeout 450 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --steps 3 --warmup 3 --e2e-steps 0 > gpurun_out/s$N.json 2> gpurun_out/s$N.err; echo s$N rc=$?
python -c "import json;d=json.load(open('gpurun_out/s$N.json'));print(d['value'],d['ms_per_step'],d['config']['rank0_ledger'])"
