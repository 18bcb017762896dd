for two in 1 0; do for fuse in 2 1; do
python -m torch.distributed.run --standalone --nproc-per-node 2 tests/summa_worker.py --sr 4 --scale 11 --grid 1x2 --fuse $fuse --mode 0 --two-round $two 2>&1 | grep -E "peak|ledger0" | sed 's/.*ledger0=//' | python -c "
import sys, ast
for l in sys.stdin:
    if 'peak_bcast_buffer_bytes_max' in l: print('two=$two fuse=$fuse', l.strip()); continue
    d = ast.literal_eval(l.strip()); print('   rank0', {k: d[k] for k in ('peak_bcast_buffer_bytes','host_bcasts','bytes_host_path','local_multiply_calls','skipped_stages')})"
done; done
