"""Local semiring SpGEMM and partial merge (the B200 hot path).

Mirrors the reference operator API:
  esc_multiply(a, b)            local_spgemm.hpp:83-156
  merge_partials(parts, r, c)   summa.hpp:122-172
  matrix_checksum(m)            checksum.hpp:20-38
but every call runs the sm_100a kernels behind the C-ABI.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import DCsr, HCsr, MultStats, check, lib
from .device import Context, DeviceCsr, default_context, hcsr_of, take_hcsr
from .formats import CscMatrix, CsrMatrix, CooMatrix, coo_to_csr


def esc_multiply(a: CsrMatrix, b: CsrMatrix, ctx: Context | None = None, stats: dict | None = None) -> CsrMatrix:
    """C = A (x) B over a.sr from HOST CSR operands (H2D + multiply + D2H).

    Same contract as the reference: ShapeError when a.ncols != b.nrows,
    result columns strictly increasing, semiring zeros dropped.
    """
    ctx = ctx or default_context()
    ha, ka = hcsr_of(a)
    hb, kb = hcsr_of(b)
    out = HCsr()
    st = MultStats()
    check(lib.spg_esc_multiply(ctx.handle, int(a.sr), C.byref(ha), C.byref(hb), C.byref(out), C.byref(st)),
          ctx.handle)
    if stats is not None:
        stats.update(st.as_dict())
    return take_hcsr(a.sr, out, False)


def local_multiply(a: DeviceCsr, b: DeviceCsr, stats: dict | None = None) -> DeviceCsr:
    """Device-resident C = A (x) B (no host traffic)."""
    out = DCsr()
    st = MultStats()
    check(lib.spg_local_multiply(a.ctx.handle, int(a.sr), C.byref(a.d), C.byref(b.d), C.byref(out),
                                 C.byref(st) if stats is not None else None), a.ctx.handle)
    if stats is not None:
        stats.update(st.as_dict())
    return DeviceCsr(a.ctx, a.sr, out)


def merge_partials(parts, block_rows: int, block_cols: int, stages=None, rounds=None,
                   stats: dict | None = None) -> DeviceCsr:
    """Merge C^T partials (DeviceCsr, block_cols x block_rows) into the CSC C block.

    Folds with SR::add in (stage, round) order and drops zeros; InternalError
    on an extents mismatch (summa.hpp:133-138).
    """
    if not parts:
        raise ValueError("merge_partials needs at least one partial to name the context")
    ctx = parts[0].ctx
    n = len(parts)
    arr = (DCsr * n)(*[p.d for p in parts])
    st_arr = (C.c_int * n)(*(stages or range(n)))
    rd_arr = (C.c_int * n)(*(rounds or [0] * n))
    out = DCsr()
    st = MultStats()
    check(lib.spg_merge_partials(ctx.handle, int(parts[0].sr), n, arr, st_arr, rd_arr, int(block_rows),
                                 int(block_cols), C.byref(out), C.byref(st) if stats is not None else None),
          ctx.handle)
    if stats is not None:
        stats.update(st.as_dict())
    return DeviceCsr(ctx, parts[0].sr, out, is_csc=True)


def matrix_checksum(m, ctx: Context | None = None) -> int:
    """matrix_checksum of a host CSR/CSC/COO or a DeviceCsr (computed on the GPU)."""
    if isinstance(m, DeviceCsr):
        return m.checksum()
    if isinstance(m, CooMatrix):
        m = coo_to_csr(m)
    d = DeviceCsr.upload(ctx or default_context(), m)
    try:
        return d.checksum()
    finally:
        d.free()
