"""Command-line front end mirroring proj/tools/spsumma.cpp.

    python -m paper_2504_06408_b200.cli multiply --gen rmat:12:16:1 --semiring tropical_i32
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 -m paper_2504_06408_b200.cli multiply ...
    python -m paper_2504_06408_b200.cli sweep --gen rmat:12:16:1 --sweep 0,65536,inf
    python -m paper_2504_06408_b200.cli verify-corpus a.mtx b.mtx

Same subcommands, flags, report layout (report.hpp:37-113: TimingReport.to_text,
sweep_table_text) and exit codes (0 ok, 1 error, 3 oracle mismatch) as the
reference CLI.  Differences, by construction of a real machine instead of a
simulated fabric:
  * --procs is the number of GPU ranks (torchrun's WORLD_SIZE; 1 without
    torchrun), laid out as the 1x1 / 1x2 / 2x2 / 2x4 grids;
  * the per-phase `sim=` column is the phase's DEVICE time (CUDA events, max
    over ranks) and `wall=` the host-measured call time split in the same
    proportions — there is no latency model to simulate;
  * the default hybrid threshold is the crossover MEASURED on the box
    (measured on the box at start-up: summa.calibrated_thresholds), the analogue
    of find_crossover(model) (tools/spsumma.cpp:186-195); --model is accepted
    and ignored;
  * --check-oracle compares against a host expand-sort-compress product of
    the input (numpy; scalar semirings, <= 4096 rows/cols as the reference's
    dense oracle limit).
"""
from __future__ import annotations

import argparse
import os
import sys
import time
import uuid

import numpy as np

from . import errors

K_INF = (1 << 64) - 1  # kInfiniteThreshold (comm.hpp)
PHASES = ("prepare", "broadcast", "local_multiply", "merge", "copy")


def parse_gen(spec: str):
    """parse_gen (tools/spsumma.cpp:33-52): rmat:<scale>:<edgefactor>:<seed>."""
    parts = spec.split(":")
    if len(parts) != 4 or parts[0] != "rmat":
        raise errors.MalformedInputError(f"--gen expects rmat:<scale>:<edgefactor>:<seed>, got '{spec}'")
    try:
        return int(parts[1]), float(parts[2]), int(parts[3])
    except ValueError:
        raise errors.MalformedInputError(f"--gen has non-numeric fields in '{spec}'") from None


def parse_comm(s: str) -> int:
    """parse_comm (tools/spsumma.cpp:54-60)."""
    from .summa import DEVICE_ONLY, HOST_ONLY, HYBRID
    modes = {"host": HOST_ONLY, "device": DEVICE_ONLY, "hybrid": HYBRID}
    if s not in modes:
        raise errors.MalformedInputError(f"--comm expects host, device, or hybrid, got '{s}'")
    return modes[s]


def parse_thresholds(text: str):
    """parse_thresholds (tools/spsumma.cpp:62-83): comma list, 'inf' allowed."""
    out = []
    for tok in text.split(","):
        if tok == "inf":
            out.append(K_INF)
        elif tok:
            try:
                out.append(int(tok))
            except ValueError:
                raise errors.MalformedInputError(f"--sweep has a non-numeric threshold '{tok}'") from None
    if not out:
        raise errors.MalformedInputError("--sweep lists no thresholds")
    return out


def fmt_threshold(t: int) -> str:
    return "inf" if t == K_INF else str(t)


def load_input(sr, matrix: str, gen: str):
    """load_input (tools/spsumma.cpp:124-134)."""
    from .generators import generate_rmat
    from .matrix_market import read_matrix_market
    if bool(matrix) == bool(gen):
        raise errors.MalformedInputError("exactly one of --matrix or --gen is required")
    if matrix:
        return read_matrix_market(sr, matrix)
    s, ef, seed = parse_gen(gen)
    return generate_rmat(sr, s, ef, seed)


def host_product(a):
    """Expand-sort-compress C = A.A on the host for --check-oracle (scalar
    semirings): products mul(a_ik, a_kj), folded per (i, j), zeros dropped."""
    from .formats import coo_to_csr
    from .semiring import SemiringId, zero
    sr = SemiringId(a.sr)
    csr = coo_to_csr(a)
    lens = np.diff(csr.rowptr)
    k_of = csr.colids
    reps = lens[k_of]
    i = np.repeat(np.repeat(np.arange(a.nrows), lens), reps)
    av = np.repeat(csr.values, reps)
    starts = np.repeat(csr.rowptr[k_of], reps)
    off = np.arange(reps.sum()) - np.repeat(np.cumsum(reps) - reps, reps)
    j = csr.colids[starts + off]
    bv = csr.values[starts + off]
    if sr == SemiringId.arithmetic:
        pv, red = av * bv, np.add
    elif sr == SemiringId.minplus:
        pv, red = av + bv, np.minimum
    elif sr == SemiringId.boolean:
        pv, red = (av & bv).astype(np.uint8), np.maximum
    elif sr == SemiringId.tropical_i32:
        inf = np.iinfo(np.int32).max
        s = av.astype(np.int64) + bv.astype(np.int64)
        s = np.clip(s, np.iinfo(np.int32).min, inf)
        s[(av == inf) | (bv == inf)] = inf
        pv, red = s.astype(np.int32), np.minimum
    else:
        raise errors.UnsupportedSemiringError("--check-oracle supports the scalar semirings only")
    order = np.lexsort((j, i))
    i, j, pv = i[order], j[order], pv[order]
    if i.size == 0:
        return i, j, pv
    key = i * a.ncols + j
    head = np.concatenate([[True], key[1:] != key[:-1]])
    idx = np.nonzero(head)[0]
    vals = red.reduceat(pv, idx)
    keep = vals != zero(sr)
    return i[idx][keep], j[idx][keep], vals[keep]


def values_close(sr, x, y) -> bool:
    """values_close (tools/spsumma.cpp:149-159): 1e-10 relative for doubles."""
    if x.dtype == np.float64:
        return bool(np.all((x == y) | (np.abs(x - y) <= 1e-10 * np.maximum(np.abs(x), np.abs(y)))))
    return x.tobytes() == y.tobytes()


def report_text(rep: dict) -> str:
    """TimingReport::to_text (report.hpp:50-98), same lines and number formats."""
    out = ["spsumma multiply report", f"matrix: {rep['matrix']}", f"semiring: {rep['semiring']}",
           f"procs: {rep['procs']}", f"comm: {rep['comm']} threshold_bytes={fmt_threshold(rep['threshold'])}",
           f"iterations: {len(rep['iterations'])} timed (after 1 untimed warm-up)",
           f"result: rows={rep['rows']} cols={rep['cols']} nnz={rep['nnz']} checksum={rep['checksum']:016x}"]
    if rep.get("oracle") is not None:
        out.append("oracle: " + ("PASS" if rep["oracle"] else "FAIL"))

    def phase_lines(tag, led):
        for p in PHASES:
            out.append(f"{tag} {p}: sim={led['sim'][p]:.9f} wall={led['wall'][p]:.9f}")
        out.append(f"{tag} payload_bcasts: host={led['host_bcasts']} device={led['device_bcasts']} "
                   f"bytes_host={led['bytes_host_path']} bytes_device={led['bytes_device_path']}")

    its = rep["iterations"]
    if its:
        out.append("first_iteration:")
        phase_lines("  first", its[0])
        mean = dict(its[0])
        mean["sim"] = {p: sum(it["sim"][p] for it in its) / len(its) for p in PHASES}
        mean["wall"] = {p: sum(it["wall"][p] for it in its) / len(its) for p in PHASES}
        out.append("mean_over_timed_iterations:")
        phase_lines("  mean", mean)
    return "\n".join(out) + "\n"


def sweep_table_text(rows) -> str:
    """sweep_table_text (report.hpp:101-113)."""
    out = ["threshold_bytes\tpct_host_bcasts\tsim_comm_seconds\twall_local_seconds\tresult_checksum"]
    for r in rows:
        out.append(f"{fmt_threshold(r['threshold'])}\t{r['pct_host']:.2f}\t{r['comm_s']:.9f}\t"
                   f"{r['local_s']:.9f}\t{r['checksum']:016x}")
    return "\n".join(out) + "\n"


class _Job:
    """One rank: process group (gloo, control plane only), grid, context, comm."""

    def __init__(self, procs: int):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", str(self.rank)))
        if procs != self.world:
            raise errors.GridError(f"--procs {procs} but {self.world} rank(s) were launched (use torchrun)")
        import torch.distributed as dist
        self.dist = dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29531")
            dist.init_process_group("gloo", rank=self.rank, world_size=self.world)
        from .device import Context
        from .summa import Comm, grid_for
        self.pr, self.pc = grid_for(self.world)
        job = [uuid.uuid4().hex[:12] if self.rank == 0 else None]
        dist.broadcast_object_list(job, src=0)
        self.ctx = Context(self.local)
        self.comm = Comm(job[0], self.world, self.rank, self.pr, self.pc, self.local)

    def max_over_ranks(self, x: float) -> float:
        import torch
        t = torch.tensor([x], dtype=torch.float64)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(self, x: int) -> int:
        import torch
        t = torch.tensor([x], dtype=torch.int64)
        self.dist.all_reduce(t)
        return int(t.item())


def _signed(x: int) -> int:
    return (x + (1 << 63)) % (1 << 64) - (1 << 63)


def _run(job, a, blk, mode, threshold, threshold_col):
    from .summa import summa25_multiply
    n = a.nrows
    job.comm.barrier()
    t0 = time.perf_counter()
    c, led = summa25_multiply(job.comm, job.ctx, blk, blk, n, a.ncols, a.ncols, mode=mode, threshold=threshold,
                              threshold_col=threshold_col, sr=a.sr)
    job.ctx.sync()
    wall = time.perf_counter() - t0
    sim = {p: job.max_over_ranks(led["ms"][p] / 1e3) for p in PHASES}
    tot = sum(sim.values()) or 1.0
    wall = job.max_over_ranks(wall)
    led = dict(led)
    led["sim"] = sim
    led["wall"] = {p: wall * sim[p] / tot for p in PHASES}
    for k in ("host_bcasts", "device_bcasts", "bytes_host_path", "bytes_device_path"):
        led[k] = job.sum_over_ranks(int(led[k]))
    return c, led


def _thresholds(job, cfg_mode, threshold):
    """Hybrid thresholds: the --threshold-bytes given, else the crossover
    measured on this box at start-up (summa.calibrated_thresholds)."""
    from .summa import HYBRID, calibrated_thresholds
    if threshold is not None:
        return threshold, threshold
    if cfg_mode != HYBRID:
        return 0, 0
    if job.world == 1:
        return 0, 0
    thr, thr_col, _ = calibrated_thresholds(job.comm, job.local, job.comm.barrier, job.max_over_ranks)
    return thr, thr_col


def cmd_multiply(args) -> int:
    from .semiring import as_id
    from .summa import checksum_part, checksum_seed, gather, local_block
    sr = as_id(args.semiring)
    mode = parse_comm(args.comm)
    job = _Job(args.procs)
    thr, thr_col = _thresholds(job, mode, args.threshold_bytes)
    a = load_input(sr, args.matrix, args.gen)
    if a.nrows != a.ncols:
        raise errors.ShapeError(f"multiply squares its input; got {a.nrows}x{a.ncols}")
    i, j = job.rank // job.pc, job.rank % job.pc
    blk = local_block(a, job.pr, job.pc, i, j)
    _run(job, a, blk, mode, thr, thr_col)  # warm-up, excluded from the report (its C is released)
    its = []
    c = None
    for _ in range(args.iters):
        c = None  # release the previous C first: its memory is reused, not mapped afresh
        c, led = _run(job, a, blk, mode, thr, thr_col)
        its.append(led)
    full = gather(job.comm, job.ctx, c, blk.rows, blk.cols, a.nrows, a.ncols, root=0)
    part = job.sum_over_ranks(_signed(checksum_part(c, blk.rows[0], blk.cols[0])))
    if job.rank != 0:
        return 0
    checksum = (checksum_seed(a.nrows, a.ncols) + (part % (1 << 64))) % (1 << 64)
    rep = {"matrix": args.matrix or args.gen, "semiring": sr.name, "procs": args.procs, "comm": args.comm,
           "threshold": thr, "rows": a.nrows, "cols": a.ncols, "nnz": full.nnz, "checksum": checksum,
           "iterations": its, "oracle": None}
    if full.checksum() != checksum:
        raise errors.InternalError("gathered C and the distributed checksum disagree")
    if args.check_oracle:
        if a.nrows > 4096 or a.ncols > 4096:
            raise errors.Error("--check-oracle refused: the dense oracle is limited to matrices of at most "
                               f"4096 rows and columns, got {a.nrows}x{a.ncols}")
        wi, wj, wv = host_product(a)
        got = full.download()  # CSC of C
        gi, gj = got.rowids, np.repeat(np.arange(a.ncols), np.diff(got.colptr))
        order = np.lexsort((gj, gi))
        rep["oracle"] = (np.array_equal(gi[order], wi) and np.array_equal(gj[order], wj)
                         and values_close(sr, got.values[order], wv))
    _emit(args.report, report_text(rep))
    return 0 if rep["oracle"] in (None, True) else 3


def cmd_sweep(args) -> int:
    """cmd_sweep (tools/spsumma.cpp:224-242) over sweep_thresholds (tuner.hpp:71-117),
    each threshold run through the real transports (comm seconds = device
    broadcast time, local seconds = multiply + merge time, max over ranks)."""
    from .semiring import as_id
    from .summa import HYBRID, checksum_part, checksum_seed, local_block
    from .tuner import default_threshold_ladder
    sr = as_id(args.semiring)
    job = _Job(args.procs)
    thresholds = (parse_thresholds(args.sweep) if args.sweep
                  else default_threshold_ladder(_thresholds(job, HYBRID, None)[0]))
    a = load_input(sr, args.matrix, args.gen)
    i, j = job.rank // job.pc, job.rank % job.pc
    blk = local_block(a, job.pr, job.pc, i, j)
    rows = []
    for t in thresholds:
        t_dev = min(int(t), (1 << 63) - 1)
        _run(job, a, blk, HYBRID, t_dev, t_dev)  # warm-up
        c, led = _run(job, a, blk, HYBRID, t_dev, t_dev)
        part = job.sum_over_ranks(_signed(checksum_part(c, blk.rows[0], blk.cols[0])))
        nb = led["host_bcasts"] + led["device_bcasts"]
        rows.append({"threshold": int(t), "pct_host": 100.0 * led["host_bcasts"] / nb if nb else 0.0,
                     "comm_s": led["sim"]["broadcast"],
                     "local_s": led["sim"]["local_multiply"] + led["sim"]["merge"],
                     "checksum": (checksum_seed(a.nrows, a.ncols) + (part % (1 << 64))) % (1 << 64)})
    if job.rank == 0:
        _emit(args.report, sweep_table_text(rows))
    return 0


def _emit(path: str, text: str):
    if not path:
        sys.stdout.write(text)
        return
    try:
        with open(path, "w") as f:
            f.write(text)
    except OSError:
        raise errors.MalformedInputError(f"{path}: cannot write report") from None


def _common(p):
    p.add_argument("--matrix", default="", help="Matrix Market coordinate file to load")
    p.add_argument("--gen", default="", help="generate input, format rmat:<scale>:<edgefactor>:<seed>")
    p.add_argument("--semiring", default="arithmetic",
                   help="arithmetic | minplus | boolean | minselect | tropical_i32 | maxtimes")
    p.add_argument("--procs", type=int, default=int(os.environ.get("WORLD_SIZE", "1")),
                   help="GPU ranks (torchrun world size)")
    p.add_argument("--comm", default="hybrid", help="host | device | hybrid")
    p.add_argument("--threshold-bytes", type=int, default=None,
                   help="hybrid routing threshold (default: crossover measured on the box)")
    p.add_argument("--model", default="", help="accepted for compatibility; curves are measured, not modelled")
    p.add_argument("--report", default="", help="write the report here instead of stdout")


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="spsumma", description="semiring SpGEMM on B200 GPUs (Sparse SUMMA)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    m = sub.add_parser("multiply", help="square a matrix and report per-phase costs")
    _common(m)
    m.add_argument("--iters", type=int, default=4, help="timed iterations (default 4)")
    m.add_argument("--check-oracle", action="store_true", help="verify the product against a host product")
    s = sub.add_parser("sweep", help="run a hybrid-threshold sweep and emit the table")
    _common(s)
    s.add_argument("--sweep", default="", help="comma-separated thresholds; 'inf' allowed")
    v = sub.add_parser("verify-corpus", help="check corpus files against their published dimensions")
    v.add_argument("files", nargs="*")
    args = ap.parse_args(argv)
    try:
        if args.cmd == "multiply":
            return cmd_multiply(args)
        if args.cmd == "sweep":
            return cmd_sweep(args)
        from .matrix_market import verify_corpus
        return verify_corpus(args.files)
    except errors.Error as e:
        sys.stderr.write(f"error: {e}\n")
        return 1


if __name__ == "__main__":
    sys.exit(main())
