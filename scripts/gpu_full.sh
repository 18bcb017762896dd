mkdir -p gpurun_out/full
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for c in 4 5 2 3; do
  timeout 2400 $TR --nproc-per-node 4 --master-port $((29700 + c)) tests/fullsize_worker.py --config $c > gpurun_out/full/c$c.out 2> gpurun_out/full/c$c.err
  echo "config $c rc=$?"; grep "\[fullsize\]" gpurun_out/full/c$c.out
done
