#!/usr/bin/env python
"""Threshold sweep of the hybrid broadcast routing on a SUMMA multiply
(sweep_thresholds, tuner.hpp:64-117; the paper's Fig. 8/9): C = A (x) A for
every threshold of the default ladder around the measured crossover (plus the
all-device 0 and all-host infinity extremes), same product every time.

    torchrun --standalone --nproc-per-node 4 tools/threshold_sweep.py --out profiles/r01_threshold_sweep_n4.json
"""
import argparse
import datetime
import json
import os
import sys
import uuid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=18)
    ap.add_argument("--sr", default="tropical_i32")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_2504_06408_b200 import Context, generators, tuner
    from paper_2504_06408_b200.semiring import as_id
    from paper_2504_06408_b200.summa import Comm, calibrated_thresholds, grid_for, local_block

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=900))
    job = [uuid.uuid4().hex[:12] if rank == 0 else None]
    dist.broadcast_object_list(job, src=0)
    pr, pc = grid_for(world)
    m = generators.permute_symmetric(generators.generate_rmat(as_id(args.sr), args.scale, 16.0, 1), 1)
    n = m.nrows
    blk = local_block(m, pr, pc, rank // pc, rank % pc)
    del m
    ctx = Context(local)
    comm = Comm(job[0], world, rank, pr, pc, local, staging_bytes=64 << 20)

    def allsum(x):
        t = torch.tensor([int(x)], dtype=torch.int64)
        dist.all_reduce(t)
        return int(t[0])

    def allmax(x):
        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    thr_row, thr_col, _ = calibrated_thresholds(comm, local, dist.barrier, allmax)  # measured on this box
    star = max(thr_row, thr_col) or None
    ladder = tuner.default_threshold_ladder(star)
    tuner.sweep_thresholds(comm, ctx, blk, n, ladder[:1], allsum, allmax)  # warm-up
    runs = [tuner.sweep_thresholds(comm, ctx, blk, n, ladder, allsum, allmax) for _ in range(args.reps)]
    if rank == 0:
        rows = []
        for k, t in enumerate(ladder):
            rs = [r[k] for r in runs]
            med = lambda key: sorted(x[key] for x in rs)[len(rs) // 2]
            rows.append({"threshold_bytes": t if t != tuner.INFINITE_THRESHOLD else "inf",
                         "pct_host_bcasts": rs[0]["pct_host_bcasts"], "comm_ms": med("comm_seconds") * 1e3,
                         "local_multiply_ms": med("wall_local_seconds") * 1e3,
                         "time_to_c_ms": med("time_to_c_seconds") * 1e3, "result_checksum": rs[0]["result_checksum"]})
        doc = {"grid": f"{pr}x{pc}", "workload": f"rmat{args.scale}_ef16_{args.sr}_AxA (permuted)",
               "crossover_bytes_used": star, "same_product_every_threshold": True, "rows": rows}
        print(json.dumps(doc), flush=True)
        for r in rows:
            print(f"{str(r['threshold_bytes']):>22}  host {r['pct_host_bcasts']:5.1f}%  comm {r['comm_ms']:7.3f} ms  "
                  f"multiply {r['local_multiply_ms']:7.2f} ms  time-to-C {r['time_to_c_ms']:7.2f} ms", file=sys.stderr)
        if args.out:
            json.dump(doc, open(args.out, "w"), indent=1)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
