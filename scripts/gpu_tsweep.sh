mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_summa.py -q -m gpu -x -k "threshold_sweep" > gpurun_out/pytest_ts.log 2>&1; echo "pytest_rc=$?"; tail -1 gpurun_out/pytest_ts.log
timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29651 --nproc-per-node 4 tools/threshold_sweep.py --out gpurun_out/threshold_sweep_n4.json > gpurun_out/tsweep4.out 2> gpurun_out/tsweep4.err; echo "n4 rc=$?"
grep -E "host|inf" gpurun_out/tsweep4.err | grep -v NCCL | tail -14
timeout 900 python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29652 --nproc-per-node 2 tools/threshold_sweep.py --out gpurun_out/threshold_sweep_n2.json > gpurun_out/tsweep2.out 2> gpurun_out/tsweep2.err; echo "n2 rc=$?"
grep -E "host|inf" gpurun_out/tsweep2.err | grep -v NCCL | tail -14
