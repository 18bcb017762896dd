set -x
N=$(nvidia-smi -L | wc -l)
export SPG_COMM_TIMEOUT_S=120 SPG_DEBUG_HANG=240 NCCL_DEBUG=WARN
for S in 12 16 18; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus $N --steps 2 --warmup 1 --scale $S > gpurun_out/summa${N}_s$S.json 2> gpurun_out/summa${N}_s$S.err; echo S=$S rc=$?
tail -c 1500 gpurun_out/summa${N}_s$S.json
done
