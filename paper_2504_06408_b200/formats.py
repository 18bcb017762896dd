"""Host sparse containers mirroring proj/include/spsumma/formats.hpp:16-86.

These are plain numpy holders (int64 indices, the reference's index width)
used at the host boundary: inputs are built here, uploaded through the C-ABI
and results come back into them.  The arithmetic never runs here.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import errors
from .semiring import as_id, dtype_of


@dataclass
class CooMatrix:
    """CooMatrix<SR> (formats.hpp:16-35): parallel tuple arrays."""

    sr: int
    nrows: int
    ncols: int
    rows: np.ndarray
    cols: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rows.shape[0])


@dataclass
class CsrMatrix:
    """CsrMatrix<SR> (formats.hpp:72-86)."""

    sr: int
    nrows: int
    ncols: int
    rowptr: np.ndarray
    colids: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.colids.shape[0])


@dataclass
class CscMatrix:
    """CscMatrix<SR> (formats.hpp:39-52)."""

    sr: int
    nrows: int
    ncols: int
    colptr: np.ndarray
    rowids: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rowids.shape[0])


@dataclass
class DcscMatrix:
    """DcscMatrix<SR> (formats.hpp:56-70): CSC with empty columns elided."""

    sr: int
    nrows: int
    ncols: int
    jc: np.ndarray
    cp: np.ndarray
    rowids: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.rowids.shape[0])


def _i64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int64))


def _vals(sr, v):
    return np.ascontiguousarray(np.asarray(v).astype(dtype_of(sr), copy=False))


def coo_to_csr(m: CooMatrix) -> CsrMatrix:
    """Row-major compression of a NORMALISED COO (unique tuples)."""
    order = np.lexsort((m.cols, m.rows))
    rows, cols, vals = m.rows[order], m.cols[order], m.values[order]
    if m.nnz and (rows.min() < 0 or rows.max() >= m.nrows or cols.min() < 0 or cols.max() >= m.ncols):
        raise errors.MalformedInputError("coo tuple outside the matrix")
    ptr = np.zeros(m.nrows + 1, dtype=np.int64)
    np.add.at(ptr, rows + 1, 1)
    return CsrMatrix(m.sr, m.nrows, m.ncols, np.cumsum(ptr), _i64(cols), _vals(m.sr, vals))


def coo_to_csc(m: CooMatrix) -> CscMatrix:
    order = np.lexsort((m.rows, m.cols))
    rows, cols, vals = m.rows[order], m.cols[order], m.values[order]
    ptr = np.zeros(m.ncols + 1, dtype=np.int64)
    np.add.at(ptr, cols + 1, 1)
    return CscMatrix(m.sr, m.nrows, m.ncols, np.cumsum(ptr), _i64(rows), _vals(m.sr, vals))


def csr_to_coo(m: CsrMatrix) -> CooMatrix:
    rows = np.repeat(np.arange(m.nrows, dtype=np.int64), np.diff(m.rowptr))
    return CooMatrix(m.sr, m.nrows, m.ncols, rows, m.colids.copy(), m.values.copy())


def csc_to_coo(m: CscMatrix) -> CooMatrix:
    cols = np.repeat(np.arange(m.ncols, dtype=np.int64), np.diff(m.colptr))
    order = np.lexsort((cols, m.rowids))
    return CooMatrix(m.sr, m.nrows, m.ncols, m.rowids[order], cols[order], m.values[order])


def csr_to_csc(m: CsrMatrix) -> CscMatrix:
    return coo_to_csc(csr_to_coo(m))


def csc_to_csr(m: CscMatrix) -> CsrMatrix:
    """csc_to_csr (formats.hpp:291-316)."""
    return coo_to_csr(csc_to_coo(m))


def reinterpret_transpose(m):
    """reinterpret_transpose (formats.hpp:255-277): zero-copy relabel."""
    if isinstance(m, CscMatrix):
        return CsrMatrix(m.sr, m.ncols, m.nrows, m.colptr, m.rowids, m.values)
    return CscMatrix(m.sr, m.ncols, m.nrows, m.rowptr, m.colids, m.values)


def csc_to_dcsc(m: CscMatrix) -> DcscMatrix:
    """csc_to_dcsc (formats.hpp:199-216)."""
    lens = np.diff(m.colptr)
    jc = np.nonzero(lens)[0].astype(np.int64)
    cp = np.concatenate([[0], m.colptr[jc + 1]]).astype(np.int64)
    return DcscMatrix(m.sr, m.nrows, m.ncols, jc, cp, m.rowids.copy(), m.values.copy())


def dcsc_decompress(m: DcscMatrix) -> CscMatrix:
    """dcsc_decompress (formats.hpp:220-250), with the reference's checks."""
    cp = m.cp
    if cp.size == 0 or cp[0] != 0 or cp.size != m.jc.size + 1 or np.any(np.diff(cp) < 0) or cp[-1] != m.nnz:
        raise errors.MalformedInputError("dcsc_decompress: bad cp offset array")
    if m.jc.size and (np.any(np.diff(m.jc) <= 0) or m.jc[0] < 0 or m.jc[-1] >= m.ncols):
        raise errors.MalformedInputError("dcsc_decompress: jc column id out of range or not strictly increasing")
    lens = np.zeros(m.ncols + 1, dtype=np.int64)
    lens[m.jc + 1] = np.diff(cp)
    return CscMatrix(m.sr, m.nrows, m.ncols, np.cumsum(lens), m.rowids.copy(), m.values.copy())


def validate(m) -> None:
    """validate (formats.hpp:335-362): offsets, strictly increasing ids, no stored zeros."""
    from .semiring import zero
    if isinstance(m, CsrMatrix):
        m = reinterpret_transpose(m)
    ptr, ids = m.colptr, m.rowids
    if ptr.size != m.ncols + 1 or ptr[0] != 0 or ptr[-1] != m.nnz or np.any(np.diff(ptr) < 0):
        raise errors.MalformedInputError("csc: offset array is not a monotone [0..nnz] map")
    seg = np.repeat(np.arange(m.ncols), np.diff(ptr))
    if ids.size:
        same = seg[1:] == seg[:-1]
        if np.any(same & (ids[1:] <= ids[:-1])) or ids.min() < 0 or ids.max() >= m.nrows:
            raise errors.MalformedInputError("csc: rows not strictly increasing")
        z = zero(m.sr)
        if np.any(m.values == z) if m.values.dtype.names is None else False:
            raise errors.MalformedInputError("csc: stored zero")
