# multi-GPU: bench line at N = all GPUs, the reference arm, and the SUMMA GPU tests on real NCCL
N=$(nvidia-smi -L | wc -l)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29540 bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/bench_n$N.json 2> gpurun_out/bench_n$N.log; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_n$N.json')); print({k: d.get(k) for k in ('value','ms_per_step','parity','n_gpus','gpu_launches')}, d['roofline']['frac'], d['config'].get('grid'), d.get('e2e'))"
timeout 900 python -m pytest tests/test_gpu_summa.py tests/test_gpu_distribute.py -x -q -m gpu > gpurun_out/gmulti_tests_n$N.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/gmulti_tests_n$N.log
