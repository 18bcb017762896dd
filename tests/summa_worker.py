"""One rank of a distributed SUMMA parity check (run under torchrun, one
process per GPU):

    torchrun --standalone --nproc-per-node N tests/summa_worker.py --sr 4 --scale 10

Each rank builds its block of A (R-MAT, identical on every rank), runs the
CUDA summa25_multiply through the C-ABI, and checks its C block bit-exactly
against the CPU oracle's product restricted to that block; the per-rank
checksum parts must add up to the oracle's matrix_checksum of the full C.
"""
import argparse
import os
import sys
import uuid

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sr", type=int, default=4)
    ap.add_argument("--scale", type=int, default=10)
    ap.add_argument("--ef", type=float, default=16.0)
    ap.add_argument("--two-round", type=int, default=1)
    ap.add_argument("--mode", type=int, default=2)
    ap.add_argument("--threshold", type=int, default=1 << 14)
    ap.add_argument("--staging", type=int, default=1 << 16)
    ap.add_argument("--fuse", type=int, default=1)
    ap.add_argument("--grid", default="", help="PRxPC (default: the BASELINE grid for the world size)")
    ap.add_argument("--gather", type=int, default=0, help="also gather C on rank 0 (GPU assembly) and compare")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--output", default="block", choices=["block", "checksum"])
    ap.add_argument("--batch-bytes", type=int, default=0)
    ap.add_argument("--golden-ledger", default="", help="golden.npz key prefix (summa_<sr>_p<p>_r<two>): compare the "
                    "distributed ledger counters with the reference's summa25_multiply")
    args = ap.parse_args()

    import torch.distributed as dist

    import oracle_bind as ob
    from paper_2504_06408_b200 import Context, generators
    from paper_2504_06408_b200.formats import coo_to_csr
    from paper_2504_06408_b200.summa import Comm, checksum_part, checksum_seed, distribute, gather, grid_for, \
        summa25_multiply

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    import torch
    local = int(os.environ.get("LOCAL_RANK", rank)) % max(1, torch.cuda.device_count())  # ranks may share a GPU
    dist.init_process_group("gloo")
    job = [uuid.uuid4().hex[:12] if rank == 0 else None]
    dist.broadcast_object_list(job, src=0)
    pr, pc = (int(x) for x in args.grid.split("x")) if args.grid else grid_for(world)
    i, j = rank // pc, rank % pc

    m = generators.generate_rmat(args.sr, args.scale, args.ef, args.seed)
    n = m.nrows
    ctx = Context(local)
    blk = distribute(ctx, m, pr, pc, only_rank=rank)  # this rank's block, built on the GPU
    comm = Comm(job[0], world, rank, pr, pc, local, staging_bytes=args.staging)
    if not comm.has_device_path and args.mode != 0:
        raise SystemExit("ranks share a GPU: run with --mode 0 (host path)")
    c, led = summa25_multiply(comm, ctx, blk, blk, n, n, n, two_round=bool(args.two_round), mode=args.mode,
                              threshold=args.threshold, fuse_stages=int(args.fuse), output=args.output,
                              batch_bytes=args.batch_bytes)
    part = checksum_part(c, blk.rows[0], blk.cols[0]) if args.output == "block" else led["checksum_part"]
    full = gather(comm, ctx, c, blk.rows, blk.cols, n, n, root=0) if args.gather else None
    got = c.download()  # CSC of the C block

    a = coo_to_csr(m)
    want_full = ob.orc_multiply(ob.Mat.of(a), ob.Mat.of(a))
    # oracle block (rows blk.rows, cols blk.cols) as CSC
    rb, re = blk.rows
    cb, ce = blk.cols
    rr = np.repeat(np.arange(n), np.diff(want_full.ptr))
    sel = (rr >= rb) & (rr < re) & (want_full.idx >= cb) & (want_full.idx < ce)
    br, bc, bv = rr[sel] - rb, want_full.idx[sel] - cb, want_full.vals[sel]
    order = np.lexsort((br, bc))
    colptr = np.concatenate([[0], np.cumsum(np.bincount(bc, minlength=ce - cb))])
    if args.output == "checksum":  # streamed: the block is not kept; nnz and checksum share are
        got.colptr, got.rowids, got.values = colptr, br[order], bv[order]
        assert led["nnz_out"] == br.size and c.nnz == 0, (led["nnz_out"], br.size, c.nnz)
        assert args.batch_bytes == 0 or led["batches"] > 1 or br.size < 64
    ok = np.array_equal(got.colptr, colptr) and np.array_equal(got.rowids, br[order])
    if args.sr == 0:  # fp64 (+, x): summation order may differ; stated tolerance 1e-12
        x, y = got.values, bv[order]
        ok = ok and bool(np.all(np.abs(x - y) <= 1e-12 * np.maximum(np.abs(x), np.abs(y)) + 1e-300))
    else:
        ok = ok and got.values.tobytes() == bv[order].tobytes()
    t = torch.tensor([part & 0xFFFFFFFF, part >> 32, int(ok), led["local_multiply_calls"],
                      led["host_bcasts"], led["device_bcasts"], led["size_exchanges"], led["skipped_stages"],
                      led["peak_bcast_buffer_bytes"]], dtype=torch.int64)
    parts = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    if rank == 0:
        total = checksum_seed(n, n)
        for p in parts:
            total = (total + int(p[0]) + (int(p[1]) << 32)) % (1 << 64)
        want = ob.orc_checksum(want_full)
        allok = all(int(p[2]) for p in parts)
        if full is not None:  # gathered full C (CSC) against the oracle's full C
            g = full.download()
            rr_all = np.repeat(np.arange(n), np.diff(want_full.ptr))
            order_all = np.lexsort((rr_all, want_full.idx))
            wcolptr = np.concatenate([[0], np.cumsum(np.bincount(want_full.idx, minlength=n))])
            gok = np.array_equal(g.colptr, wcolptr) and np.array_equal(g.rowids, rr_all[order_all])
            if args.sr == 0:
                x, y = g.values, want_full.vals[order_all]
                gok = gok and bool(np.all(np.abs(x - y) <= 1e-12 * np.maximum(np.abs(x), np.abs(y)) + 1e-300))
            else:
                gok = gok and g.values.tobytes() == want_full.vals[order_all].tobytes()
            print(f"[summa_worker] gather_ok={gok}", flush=True)
            allok = allok and gok
        cs_ok = total == want or args.sr == 0  # fp64 values hash bitwise
        if args.golden_ledger:
            # the reference charges each collective once (fabric.hpp:220-241); every rank of a
            # square q x q grid counts the q-rank collectives it joins, and its own multiplies
            g = np.load(os.path.join(HERE, "golden", "golden.npz"))
            gl = g[args.golden_ledger + "_ledger"]
            q = pr
            bc = sum(int(p[4]) + int(p[5]) for p in parts)
            sx = sum(int(p[6]) for p in parts)
            lm = sum(int(p[3]) for p in parts)
            sk = sum(int(p[7]) for p in parts)
            led_ok = (pr == pc and bc == q * (gl[0] + gl[1]) and sx == q * gl[4] and sk == gl[6]
                      and (args.fuse or lm == gl[5]))
            led_ok = led_ok and total == int(g[args.golden_ledger + "_csum"][0])
            print(f"[summa_worker] golden ledger {args.golden_ledger}: bcasts {bc}/{q} vs {gl[0] + gl[1]}, "
                  f"size exchanges {sx}/{q} vs {gl[4]}, multiplies {lm} vs {gl[5]}, skipped {sk} vs {gl[6]}: "
                  f"ledger_ok={led_ok}", flush=True)
            allok = allok and led_ok
        print(f"[summa_worker] peak_bcast_buffer_bytes_max={max(int(p[8]) for p in parts)}", flush=True)
        print(f"[summa_worker] grid {pr}x{pc} sr={args.sr} s{args.scale} two_round={args.two_round} "
              f"mode={args.mode} fuse={args.fuse}: blocks_ok={allok} checksum_ok={cs_ok} ledger0={led}", flush=True)
        if not (allok and cs_ok):
            sys.exit(1)
    comm.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
