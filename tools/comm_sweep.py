#!/usr/bin/env python
"""Measured hybrid-communication sweep (BASELINE config 5's "hybrid-comm
threshold sweep 1 KB-1 GB"; paper Fig. 7-9).

Run one process per GPU on a 1 x N grid (the row scope has fanout N):

    torchrun --standalone --nproc-per-node 2 tools/comm_sweep.py --out profiles/comm_fanout2.json
    torchrun --standalone --nproc-per-node 4 tools/comm_sweep.py --out profiles/comm_fanout4.json

For every size 2^10 .. 2^30 bytes it times the host path (pinned shared-memory
staging) and the device path (NCCL over NVLink) through spg_bcast, finds the
crossover with the reference's bisection (tuner.hpp:17-39), then times the
HYBRID path at that threshold and checks hybrid <= min(host, device) per size
(within noise) and in aggregate.  Rank 0 writes the curves in the reference's
latency-model JSON format plus the verdict.
"""
import argparse
import datetime
import json
import os
import sys
import time
import uuid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log2", type=int, default=10)
    ap.add_argument("--max-log2", type=int, default=30)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    from paper_2504_06408_b200 import tuner
    from paper_2504_06408_b200.summa import HYBRID, Comm

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=600))
    job = [uuid.uuid4().hex[:12] if rank == 0 else None]
    dist.broadcast_object_list(job, src=0)
    comm = Comm(job[0], world, rank, 1, world, local, staging_bytes=64 << 20)

    def reduce_max(x):
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    sizes = [1 << k for k in range(args.min_log2, args.max_log2 + 1)]
    curves = tuner.measure_bcast_curves(comm, sizes, reps=args.reps, scope=0, barrier=dist.barrier,
                                        reduce_max=reduce_max, device=local, fanout=world)
    host, dev = curves["host_path_total"], curves["device_path_total"]
    xo = tuner.find_crossover(host, dev, sizes[0], sizes[-1])
    thr = xo if xo is not None else (sizes[-1] + 1 if host[-1][1] < dev[-1][1] else 0)

    # hybrid at the measured threshold, same protocol
    buf = torch.empty(sizes[-1], dtype=torch.uint8, device=f"cuda:{local}")
    hybrid = []
    for nbytes in sizes:
        ts = []
        for r in range(args.reps + 2):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            comm.bcast(0, 0, buf.data_ptr(), nbytes, mode=HYBRID, threshold=thr)
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(time.perf_counter() - t0)
        hybrid.append((float(nbytes), reduce_max(sorted(ts)[len(ts) // 2])))

    if rank == 0:
        rows = []
        ok_all = True
        for (b, h), (_, d), (_, y) in zip(host, dev, hybrid):
            best = min(h, d)
            ok = y <= best * 1.15 + 5e-6  # within noise of the better pure path
            ok_all &= ok
            rows.append({"bytes": int(b), "host_s": h, "device_s": d, "hybrid_s": y, "hybrid_le_min": ok})
        agg = {"host_only_s": sum(h for _, h in host), "device_only_s": sum(d for _, d in dev),
               "hybrid_s": sum(y for _, y in hybrid)}
        verdict = {"fanout": world, "crossover_bytes": xo, "threshold_used": thr, "rows": rows,
                   "aggregate": agg, "hybrid_le_min_every_size": ok_all,
                   "hybrid_beats_both_in_aggregate": agg["hybrid_s"] < min(agg["host_only_s"], agg["device_only_s"])}
        print(json.dumps({k: v for k, v in verdict.items() if k != "rows"}), flush=True)
        for r in rows:
            print(f"{r['bytes']:>12d}  host {r['host_s'] * 1e6:10.1f} us  device {r['device_s'] * 1e6:10.1f} us  "
                  f"hybrid {r['hybrid_s'] * 1e6:10.1f} us  {'ok' if r['hybrid_le_min'] else 'SLOW'}",
                  file=sys.stderr)
        if args.out:
            tuner.save_model(args.out, curves, extra={"sweep": verdict}, fanout=world)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
