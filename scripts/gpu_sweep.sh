set -x
export SPG_COMM_TIMEOUT_S=120
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 2 tools/comm_sweep.py --out gpurun_out/comm_fanout2.json > gpurun_out/sweep2.out 2> gpurun_out/sweep2.err; echo rc=$?
cat gpurun_out/sweep2.out; grep -E "host .*device" gpurun_out/sweep2.err
timeout 600 python -m torch.distributed.run --standalone --nproc-per-node 4 tools/comm_sweep.py --out gpurun_out/comm_fanout4.json > gpurun_out/sweep4.out 2> gpurun_out/sweep4.err; echo rc=$?
cat gpurun_out/sweep4.out; grep -E "host .*device" gpurun_out/sweep4.err
