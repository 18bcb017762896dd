"""Synthetic workloads of the BASELINE configs (host C++ behind the C-ABI).

generate_rmat is bit-identical to the reference generator (rmat.hpp:15-60);
generate_er / generate_stencil27 are the config-5 / config-4 inputs
(SURVEY.md §8d).  All return normalised COO (row-major, unique).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib
from .formats import CooMatrix, CsrMatrix, CscMatrix
from .semiring import as_id, dtype_of


def _take(sr, nnz, rows, cols, vals):
    n = int(nnz)
    dt = dtype_of(sr)
    r = np.ctypeslib.as_array(rows, shape=(max(n, 1),))[:n].copy()
    c = np.ctypeslib.as_array(cols, shape=(max(n, 1),))[:n].copy()
    from .device import copy_out
    v = copy_out(vals, n, dt)
    lib.spg_free(C.cast(rows, C.c_void_p))
    lib.spg_free(C.cast(cols, C.c_void_p))
    lib.spg_free(vals)
    return r, c, v


def generate_rmat(sr, scale: int, edge_factor: float, seed: int) -> CooMatrix:
    sr = as_id(sr)
    nrows, nnz = C.c_int64(), C.c_int64()
    rows, cols = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
    vals = C.c_void_p()
    check(lib.spg_generate_rmat(int(sr), int(scale), float(edge_factor), int(seed), C.byref(nrows),
                                C.byref(nnz), C.byref(rows), C.byref(cols), C.byref(vals)))
    r, c, v = _take(sr, nnz.value, rows, cols, vals)
    return CooMatrix(int(sr), nrows.value, nrows.value, r, c, v)


def generate_er(sr, n: int, d: int, seed: int, value_mode: int = 0) -> CooMatrix:
    sr = as_id(sr)
    nnz = C.c_int64()
    rows, cols = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
    vals = C.c_void_p()
    check(lib.spg_generate_er(int(sr), int(n), int(d), int(seed), int(value_mode), C.byref(nnz),
                              C.byref(rows), C.byref(cols), C.byref(vals)))
    r, c, v = _take(sr, nnz.value, rows, cols, vals)
    return CooMatrix(int(sr), int(n), int(n), r, c, v)


def generate_stencil27(sr, N: int) -> CooMatrix:
    sr = as_id(sr)
    nrows, nnz = C.c_int64(), C.c_int64()
    rows, cols = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
    vals = C.c_void_p()
    check(lib.spg_generate_stencil27(int(sr), int(N), C.byref(nrows), C.byref(nnz), C.byref(rows),
                                     C.byref(cols), C.byref(vals)))
    r, c, v = _take(sr, nnz.value, rows, cols, vals)
    return CooMatrix(int(sr), nrows.value, nrows.value, r, c, v)


def generate_er_block(sr, n: int, d: int, seed: int, rows: tuple, cols: tuple, value_mode: int = 0) -> CooMatrix:
    """Block rows[0]:rows[1] x cols[0]:cols[1] of generate_er, LOCAL indices."""
    sr = as_id(sr)
    nnz = C.c_int64()
    r_, c_ = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
    vals = C.c_void_p()
    check(lib.spg_generate_er_block(int(sr), int(n), int(d), int(seed), int(value_mode), int(rows[0]), int(rows[1]),
                                    int(cols[0]), int(cols[1]), C.byref(nnz), C.byref(r_), C.byref(c_),
                                    C.byref(vals)))
    r, c, v = _take(sr, nnz.value, r_, c_, vals)
    return CooMatrix(int(sr), rows[1] - rows[0], cols[1] - cols[0], r - rows[0], c - cols[0], v)


def generate_stencil27_block(sr, N: int, rows: tuple, cols: tuple) -> CooMatrix:
    """Block of generate_stencil27 with LOCAL indices."""
    sr = as_id(sr)
    nrows, nnz = C.c_int64(), C.c_int64()
    r_, c_ = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
    vals = C.c_void_p()
    check(lib.spg_generate_stencil27_block(int(sr), int(N), int(rows[0]), int(rows[1]), int(cols[0]), int(cols[1]),
                                           C.byref(nrows), C.byref(nnz), C.byref(r_), C.byref(c_), C.byref(vals)))
    r, c, v = _take(sr, nnz.value, r_, c_, vals)
    return CooMatrix(int(sr), rows[1] - rows[0], cols[1] - cols[0], r - rows[0], c - cols[0], v)


def coo_to_csr_fast(m: CooMatrix, to_csc: bool = False):
    """Compression of a normalised COO with the library's host routine."""
    from ._lib import HCsr
    from .device import take_hcsr
    rows = np.ascontiguousarray(m.rows, dtype=np.int64)
    cols = np.ascontiguousarray(m.cols, dtype=np.int64)
    vals = np.ascontiguousarray(m.values)
    out = HCsr()
    check(lib.spg_coo_to_csr(int(m.sr), int(m.nrows), int(m.ncols), int(m.nnz),
                             rows.ctypes.data_as(C.POINTER(C.c_int64)), cols.ctypes.data_as(C.POINTER(C.c_int64)),
                             vals.ctypes.data_as(C.c_void_p), int(to_csc), C.byref(out)))
    return take_hcsr(m.sr, out, to_csc)


def permute_symmetric(m: CooMatrix, seed: int) -> CooMatrix:
    """Relabel vertices by a seeded random permutation p: A' = P A P^T
    (entry (i, j) -> (p[i], p[j])), re-normalised row-major.  Work and output
    size of A'.A' equal those of A.A; CombBLAS applies the same relabeling to
    balance R-MAT blocks across a process grid."""
    if m.nrows != m.ncols:
        raise ValueError("symmetric permutation needs a square matrix")
    perm = np.random.default_rng(seed).permutation(m.nrows).astype(np.int64)
    r, c = perm[m.rows], perm[m.cols]
    order = np.lexsort((c, r))
    return CooMatrix(m.sr, m.nrows, m.ncols, r[order], c[order], m.values[order])
