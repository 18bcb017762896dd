#!/usr/bin/env python
"""Local multiply probe: C = A.A for one generated matrix on cuda:0, per-bin
row counts and phase times (spg_mult_stats), repeated --reps times.

    python tools/local_probe.py er --n-log2 16 --d 64 --sr maxtimes --value-mode 1
    python tools/local_probe.py stencil --N 120 --sr arithmetic
    python tools/local_probe.py rmat --scale 18 --sr tropical_i32
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("kind", choices=["er", "stencil", "rmat"])
    ap.add_argument("--n-log2", type=int, default=16)
    ap.add_argument("--d", type=int, default=64)
    ap.add_argument("--N", type=int, default=100)
    ap.add_argument("--scale", type=int, default=16)
    ap.add_argument("--sr", default="maxtimes")
    ap.add_argument("--value-mode", type=int, default=0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--permute", action="store_true")
    ap.add_argument("--block", type=int, nargs=4, default=None, metavar=("PR", "PC", "I", "J"),
                    help="multiply block row I of A by block column J of A (the local work of grid rank (I, J))")
    ap.add_argument("--frange", type=float, nargs=2, default=None,
                    help="keep only rows of the left operand whose product count F is in (lo, hi]")
    args = ap.parse_args()
    from paper_2504_06408_b200 import Context, DeviceCsr, generators, local_multiply
    from paper_2504_06408_b200.semiring import as_id

    sr = as_id(args.sr)
    t0 = time.time()
    if args.kind == "er":
        coo = generators.generate_er(sr, 1 << args.n_log2, args.d, 1, value_mode=args.value_mode)
    elif args.kind == "stencil":
        coo = generators.generate_stencil27(sr, args.N)
    else:
        coo = generators.generate_rmat(sr, args.scale, 16.0, 1)
    if args.permute:
        coo = generators.permute_symmetric(coo, 1)
    a = generators.coo_to_csr_fast(coo)
    print(f"gen {time.time() - t0:.1f}s n={a.nrows} nnz={a.nnz}", file=sys.stderr)
    import numpy as np
    from paper_2504_06408_b200.formats import CsrMatrix
    left = a
    if args.frange:
        rl = np.diff(a.rowptr)
        F = np.zeros(a.nrows, np.int64)
        np.add.at(F, np.repeat(np.arange(a.nrows), rl), rl[a.colids])
        keep = np.nonzero((F > args.frange[0]) & (F <= args.frange[1]))[0]
        lens = rl[keep]
        ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        sel = np.concatenate([np.arange(a.rowptr[r], a.rowptr[r + 1]) for r in keep]) if keep.size else np.zeros(0, np.int64)
        left = CsrMatrix(a.sr, keep.size, a.ncols, ptr, a.colids[sel], a.values[sel])
        print(f"rows with F in ({args.frange[0]:.0f}, {args.frange[1]:.0f}]: {keep.size}, products {F[keep].sum()}",
              file=sys.stderr)
    right = a
    if args.block:
        from paper_2504_06408_b200.summa import block_range
        pr, pc, bi, bj = args.block
        r0, r1 = block_range(a.nrows, pr, bi)
        c0, c1 = block_range(a.ncols, pc, bj)
        rows_ = np.arange(r0, r1)
        lens = np.diff(a.rowptr)[r0:r1]
        left = CsrMatrix(a.sr, r1 - r0, a.ncols, np.concatenate([[0], np.cumsum(lens)]).astype(np.int64),
                         a.colids[a.rowptr[r0]:a.rowptr[r1]], a.values[a.rowptr[r0]:a.rowptr[r1]])
        keep = (a.colids >= c0) & (a.colids < c1)
        rr = np.repeat(np.arange(a.nrows), np.diff(a.rowptr))[keep]
        ptr = np.concatenate([[0], np.cumsum(np.bincount(rr, minlength=a.nrows))]).astype(np.int64)
        right = CsrMatrix(a.sr, a.nrows, c1 - c0, ptr, a.colids[keep] - c0, a.values[keep])
        print(f"block ({bi},{bj}) of {pr}x{pc}: left {left.nrows}x{left.ncols} nnz {left.nnz}, right nnz {right.nnz}",
              file=sys.stderr)
    ctx = Context(0)
    d = DeviceCsr.upload(ctx, right)
    dl = DeviceCsr.upload(ctx, left) if left is not a else DeviceCsr.upload(ctx, a)
    for r in range(args.reps):
        st = {}
        c = local_multiply(dl, d, stats=st)
        ctx.sync()
        print(json.dumps({"rep": r, **st}))
        c.free()


if __name__ == "__main__":
    main()
