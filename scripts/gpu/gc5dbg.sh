export SPG_HOST_TRACE=20
timeout 900 python bench.py --config 5 --summa --gpus 1 --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > /dev/null 2> gpurun_out/c5dbg_n1.log; echo n1 rc=$?
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --config 5 --gpus 2 --steps 1 --warmup 3 --e2e-steps 0 > /dev/null 2> gpurun_out/c5dbg_n2.log; echo n2 rc=$?
grep "summa batch" gpurun_out/c5dbg_n1.log | tail -9
grep "summa batch\|cudaMalloc" gpurun_out/c5dbg_n2.log | tail -30
