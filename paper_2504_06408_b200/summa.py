"""Distributed Sparse SUMMA (2.5D) over one process per B200.

Mirrors summa25_multiply (proj/include/spsumma/summa.hpp:248-349) with the
reference's DistMatrix (dist_matrix.hpp:41-141) generalised from q x q to
pr x pc grids.  The per-rank program, the broadcasts and the merge run in
C++/CUDA behind the C-ABI (spg_summa25_multiply); this module only builds
the host blocks and calls it.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import errors
from ._lib import DCsr, HCsr, HDcsc, Ledger, SummaOpts, check, lib
from .device import Context, DeviceCsr, hcsr_of
from .formats import CooMatrix, CscMatrix, DcscMatrix, coo_to_csc, csc_to_dcsc
from .semiring import as_id

HOST_ONLY, DEVICE_ONLY, HYBRID = 0, 1, 2
GRIDS = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}


def grid_for(world: int):
    """pr x pc for the BASELINE GPU counts (1x1, 1x2, 2x2, 2x4); otherwise the
    most square factorisation with pr <= pc."""
    if world in GRIDS:
        return GRIDS[world]
    pr = int(np.floor(np.sqrt(world)))
    while world % pr:
        pr -= 1
    return pr, world // pr


def block_range(n: int, q: int, idx: int):
    """block_range (dist_matrix.hpp:23-28): larger ranges first."""
    b, e = C.c_int64(), C.c_int64()
    lib.spg_block_range(int(n), int(q), int(idx), C.byref(b), C.byref(e))
    return b.value, e.value


@dataclass
class LocalBlock:
    """LocalBlock (dist_matrix.hpp:41-53): CSC or DCSC storage + extents."""

    storage: object  # CscMatrix | DcscMatrix
    rows: tuple
    cols: tuple

    @property
    def is_dcsc(self):
        return isinstance(self.storage, DcscMatrix)


def local_block(m: CooMatrix, pr: int, pc: int, i: int, j: int) -> LocalBlock:
    """Block (i, j) of `m` on a pr x pc grid, stored DCSC when fewer than half
    of its columns are populated (distribute, dist_matrix.hpp:69-111)."""
    rb, re = block_range(m.nrows, pr, i)
    cb, ce = block_range(m.ncols, pc, j)
    sel = (m.rows >= rb) & (m.rows < re) & (m.cols >= cb) & (m.cols < ce)
    piece = CooMatrix(m.sr, re - rb, ce - cb, m.rows[sel] - rb, m.cols[sel] - cb, m.values[sel])
    return block_from_piece(piece, (rb, re), (cb, ce))


def distribute(ctx: Context, m: CooMatrix, pr: int, pc: int, only_rank: int | None = None):
    """distribute (dist_matrix.hpp:69-111) on the GPU (spg_distribute): the
    COO is uploaded once, routed to its blocks, sorted column-major per block
    by one device radix sort, duplicates folded with SR::add in input order
    and zeros dropped (coo_to_csc, formats.hpp:138-180); a block with fewer
    than half of its columns populated comes back DCSC.  Returns the list of
    pr * pc LocalBlocks (rank = i * pc + j), or only `only_rank`'s block."""
    from ._lib import Block
    from .device import copy_out
    from .semiring import dtype_of
    rows = np.ascontiguousarray(m.rows, dtype=np.int64)
    cols = np.ascontiguousarray(m.cols, dtype=np.int64)
    vals = np.ascontiguousarray(m.values, dtype=dtype_of(m.sr))
    n = 1 if only_rank is not None else pr * pc
    out = (Block * n)()
    i64 = C.POINTER(C.c_int64)
    check(lib.spg_distribute(ctx.handle, int(m.sr), int(m.nrows), int(m.ncols), int(rows.shape[0]),
                             rows.ctypes.data_as(i64), cols.ctypes.data_as(i64), vals.ctypes.data_as(C.c_void_p),
                             int(pr), int(pc), -1 if only_rank is None else int(only_rank), out), ctx.handle)
    dt = dtype_of(m.sr)
    blocks = []
    try:
        for b in out:
            if b.is_dcsc:
                d = b.dcsc
                st = DcscMatrix(m.sr, d.nrows, d.ncols, copy_out(d.jc, d.njc, np.int64),
                                copy_out(d.cp, d.njc + 1, np.int64), copy_out(d.rowids, d.nnz, np.int64),
                                copy_out(d.vals, d.nnz, dt))
            else:
                h = b.csc
                st = CscMatrix(m.sr, h.nrows, h.ncols, copy_out(h.ptr, h.ncols + 1, np.int64),
                               copy_out(h.idx, h.nnz, np.int64), copy_out(h.vals, h.nnz, dt))
            blocks.append(LocalBlock(st, (b.row_begin, b.row_end), (b.col_begin, b.col_end)))
    finally:
        for b in out:
            lib.spg_block_free(C.byref(b))
    return blocks[0] if only_rank is not None else blocks


def block_from_piece(piece: CooMatrix, rows: tuple, cols: tuple) -> LocalBlock:
    """LocalBlock from a block's COO in LOCAL indices (e.g. the block
    generators), DCSC when fewer than half of its columns are populated.
    `piece` must be normalised (row-major sorted, unique)."""
    from .generators import coo_to_csr_fast
    csc = coo_to_csr_fast(piece, to_csc=True)
    populated = int(np.count_nonzero(np.diff(csc.colptr)))
    storage = csc_to_dcsc(csc) if 2 * populated < csc.ncols else csc
    return LocalBlock(storage, tuple(rows), tuple(cols))


def _block_structs(blk: LocalBlock):
    s = blk.storage
    if isinstance(s, DcscMatrix):
        jc = np.ascontiguousarray(s.jc, dtype=np.int64)
        cp = np.ascontiguousarray(s.cp, dtype=np.int64)
        ri = np.ascontiguousarray(s.rowids, dtype=np.int64)
        v = np.ascontiguousarray(s.values)
        d = HDcsc(s.nrows, s.ncols, ri.shape[0], jc.shape[0], jc.ctypes.data_as(C.POINTER(C.c_int64)),
                  cp.ctypes.data_as(C.POINTER(C.c_int64)), ri.ctypes.data_as(C.POINTER(C.c_int64)),
                  v.ctypes.data_as(C.c_void_p))
        return None, d, (jc, cp, ri, v)
    h, keep = hcsr_of(s)
    return h, None, keep


class Comm:
    """spg_comm: shared-memory rendezvous + pinned staging + NCCL row/column
    communicators for one rank of a pr x pc grid (rank = i * pc + j)."""

    def __init__(self, job: str, world: int, rank: int, pr: int, pc: int, device: int,
                 staging_bytes: int = 64 << 20):
        h = C.c_void_p()
        rc = lib.spg_comm_create(job.encode(), world, rank, pr, pc, device, staging_bytes, C.byref(h))
        if rc != 0:
            raise errors.from_status(rc, lib.spg_comm_last_error(None).decode())
        self.handle, self.world, self.rank, self.pr, self.pc = h, world, rank, pr, pc
        self.row, self.col = rank // pc, rank % pc

    def _check(self, rc):
        if rc != 0:
            raise errors.from_status(rc, lib.spg_comm_last_error(self.handle).decode())

    @property
    def has_device_path(self) -> bool:
        """False when ranks share a GPU (no NCCL communicator): host path only."""
        return bool(lib.spg_comm_has_device_path(self.handle))

    def barrier(self):
        self._check(lib.spg_comm_barrier(self.handle))

    def exchange_sizes(self, scope: int, root: int, triple):
        """Rank::exchange_sizes (fabric.hpp:335-338); scope 0 = grid row, 1 = column."""
        t = (C.c_int64 * 3)(*triple)
        self._check(lib.spg_exchange_sizes(self.handle, scope, root, t))
        return tuple(t)

    def bcast(self, scope: int, root: int, ptr: int, nbytes: int, mode: int = HYBRID, threshold: int = 0) -> int:
        """Rank::bcast (fabric.hpp:343-349) of a device (or host) buffer; returns the path taken."""
        path = C.c_int()
        self._check(lib.spg_bcast(self.handle, scope, root, C.c_void_p(ptr), int(nbytes), mode, int(threshold),
                                  C.byref(path)))
        return path.value

    def set_device_transport(self, transport: int):
        self._check(lib.spg_comm_set_device_transport(self.handle, transport))

    def close(self):
        if self.handle:
            lib.spg_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def summa25_multiply(comm: Comm, ctx: Context, a_block: LocalBlock, b_block: LocalBlock, a_nrows: int,
                     a_ncols: int, b_ncols: int, two_round: bool = True, mode: int = HYBRID,
                     threshold: int = 0, sr=None, fuse_stages: bool = True, threshold_col: int = 0,
                     output: str = "block", batch_bytes: int = 0):
    """One rank's summa25_multiply.  Returns (C block as DeviceCsr CSC, ledger dict).

    fuse_stages=True (1) keeps every received panel and runs one fused local
    multiply over the concatenated panels (no partials, no merge); 2 fuses per
    2.5D round and folds the round products with the GPU merge (only one
    round's panels resident: the 2.5D memory bound); False (0) runs the
    reference's per-stage multiplies followed by merge_partials.
    output="checksum" streams a C block larger than HBM: the fused multiply
    runs in column batches (<= batch_bytes of C each), each batch is
    checksummed and released; ledger["checksum_part"] / ["nnz_out"] carry the
    block's share and the returned block is empty."""
    sr = as_id(sr if sr is not None else a_block.storage.sr)
    ah, ad, ka = _block_structs(a_block)
    bh, bd, kb = _block_structs(b_block)
    opts = SummaOpts(int(two_round), int(mode), int(threshold), int(threshold_col), int(fuse_stages),
                     {"block": 0, "checksum": 1}[output], int(batch_bytes))
    out = DCsr()
    led = Ledger()
    rc = lib.spg_summa25_multiply(comm.handle, ctx.handle, int(sr), int(a_nrows), int(a_ncols), int(b_ncols),
                                  C.byref(ah) if ah is not None else None, C.byref(ad) if ad is not None else None,
                                  C.byref(bh) if bh is not None else None, C.byref(bd) if bd is not None else None,
                                  C.byref(opts), C.byref(out), C.byref(led))
    check(rc, ctx.handle)
    return DeviceCsr(ctx, sr, out, is_csc=True), led.as_dict()


def gather(comm: Comm, ctx: Context, c_block: DeviceCsr, rows: tuple, cols: tuple, nrows: int, ncols: int,
           root: int = 0):
    """gather (dist_matrix.hpp): this rank's CSC block of C
    (global extents rows/cols) to world rank `root`, assembled on its GPU.
    Collective; returns the full CSC DeviceCsr on the root, None elsewhere."""
    out = DCsr()
    check(lib.spg_gather(comm.handle, ctx.handle, int(c_block.sr), C.byref(c_block.d), int(rows[0]), int(cols[0]),
                         int(nrows), int(ncols), int(root), C.byref(out)), ctx.handle)
    if comm.rank != root:
        return None
    return DeviceCsr(ctx, c_block.sr, out, is_csc=True)


def checksum_part(c: DeviceCsr, row_off: int, col_off: int) -> int:
    """This block's share of matrix_checksum of the distributed matrix."""
    out = C.c_uint64()
    check(lib.spg_checksum_part(c.ctx.handle, int(c.sr), C.byref(c.d), int(c.is_csc), int(row_off), int(col_off),
                                C.byref(out)), c.ctx.handle)
    return int(out.value)


def checksum_seed(nrows: int, ncols: int) -> int:
    return int(lib.spg_checksum_seed(int(nrows), int(ncols)))


def calibrated_thresholds(comm: "Comm", device: int, barrier, reduce_max, reps: int = 5) -> tuple:
    """(row-scope, column-scope) hybrid thresholds MEASURED on this box at
    start-up (tuner.calibrate_threshold over the real transports; cached per
    GPU model and grid): the row scope has fanout pc, the column scope pr.
    Collective over all ranks.  Returns (thr_row, thr_col, info)."""
    import torch

    from . import tuner
    name = torch.cuda.get_device_name(device).replace(" ", "_")
    key = f"{name}_{comm.pr}x{comm.pc}"
    out, info = [], {}
    for scope, fanout in ((0, comm.pc), (1, comm.pr)):
        if fanout < 2:  # a one-rank scope never broadcasts
            out.append(0)
            info[("row", "col")[scope]] = {"threshold": 0, "source": "one-rank scope"}
            continue
        cal = tuner.calibrate_threshold(comm, scope, fanout, device, barrier, reduce_max, reps=reps, cache_key=key)
        out.append(int(cal["threshold"]))
        info[("row", "col")[scope]] = cal
    return out[0], out[1], info


def measured_threshold(fanout: int, default: int = 64 << 10) -> int:
    """Offline reference point only (tools / docs): the crossover recorded by
    tools/comm_sweep.py in profiles/comm_fanout<f>.json on an earlier box.
    The product path measures its threshold on the running box instead
    (calibrated_thresholds)."""
    import json
    import os
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
    best = None
    for f in os.listdir(root) if os.path.isdir(root) else []:
        if f.startswith("comm_fanout") and f.endswith(".json"):
            try:
                k = int(f[len("comm_fanout"):-len(".json")])
                x = json.load(open(os.path.join(root, f)))["sweep"]["crossover_bytes"]
            except (ValueError, KeyError, OSError):
                continue
            if x and (best is None or abs(k - fanout) < abs(best[0] - fanout)):
                best = (k, int(x))
    return best[1] if best else default
