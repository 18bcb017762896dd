"""ctypes bindings to the TEST-ONLY checkers under oracle/.

  oracle/liboracle.so            CPU restatement (Gustavson SPA) — the parity oracle
  oracle/_ref/libspsumma_ref.so  the unmodified reference compiled from its headers

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module; the product path never does.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libspsumma_ref.so")

_DT = {0: np.dtype("<f8"), 1: np.dtype("<f8"), 2: np.dtype("u1"),
       3: np.dtype([("weight", "<f8"), ("payload", "<i8")]), 4: np.dtype("<i4"),
       5: np.dtype([("w", "<f8"), ("tag", "<u8")])}


class Csr(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("ptr", C.POINTER(C.c_int64)), ("idx", C.POINTER(C.c_int64)), ("vals", C.c_void_p)]


class Coo(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("rows", C.POINTER(C.c_int64)), ("cols", C.POINTER(C.c_int64)), ("vals", C.c_void_p)]


def _load(path):
    if not os.path.exists(path):
        return None
    return C.CDLL(path)


orc = _load(ORACLE_SO)
ref = _load(REF_SO)
_P = C.POINTER
if orc is not None:
    orc.orc_multiply.argtypes = [C.c_int, _P(Csr), _P(Csr), C.c_int, _P(Csr)]
    orc.orc_multiply_stream.argtypes = [C.c_int, _P(Csr), _P(Csr), C.c_int64, C.c_int64, C.c_int,
                                        _P(C.c_uint64), _P(C.c_int64), _P(C.c_int64), _P(C.c_int64)]
    orc.orc_checksum.argtypes = [C.c_int, _P(Csr), C.c_int, _P(C.c_uint64)]
    orc.orc_checksum_seed.restype = C.c_uint64
    orc.orc_checksum_seed.argtypes = [C.c_int64, C.c_int64]
    orc.orc_free.argtypes = [C.c_void_p]
if ref is not None:
    ref.ref_last_error.restype = C.c_char_p
    ref.ref_free.argtypes = [C.c_void_p]
    ref.ref_generate_rmat.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, _P(Coo)]
    ref.ref_read_matrix_market.argtypes = [C.c_int, C.c_char_p, _P(Coo)]
    ref.ref_random_coo.argtypes = [C.c_int, C.c_uint64, C.c_int64, C.c_int64, C.c_double, C.c_int, _P(Coo)]
    ref.ref_esc_multiply.argtypes = [C.c_int, _P(Csr), _P(Csr), C.c_uint64, _P(Csr)]
    ref.ref_naive_multiply.argtypes = [C.c_int, _P(Csr), _P(Csr), _P(Csr)]
    ref.ref_coo_to_csr.argtypes = [C.c_int, _P(Coo), _P(Csr)]
    ref.ref_coo_to_csc.argtypes = [C.c_int, _P(Coo), _P(Csr)]
    ref.ref_checksum_csr.argtypes = [C.c_int, _P(Csr), _P(C.c_uint64)]
    ref.ref_checksum_csc.argtypes = [C.c_int, _P(Csr), _P(C.c_uint64)]
    ref.ref_csr_slice.argtypes = [C.c_int, _P(Csr), C.c_int, C.c_int64, C.c_int64, _P(Csr)]
    ref.ref_merge_partials.argtypes = [C.c_int, C.c_int, _P(Csr), _P(C.c_int), _P(C.c_int), C.c_int64,
                                       C.c_int64, _P(Csr)]
    ref.ref_block_range.argtypes = [C.c_int64, C.c_int, C.c_int, _P(C.c_int64), _P(C.c_int64)]
    ref.ref_round_range.argtypes = [C.c_int64, C.c_int, C.c_int, _P(C.c_int64), _P(C.c_int64)]
    ref.ref_dcsc_roundtrip.argtypes = [C.c_int, _P(Csr), _P(C.c_int64), _P(Csr)]
    ref.ref_distribute_block.argtypes = [C.c_int, _P(Coo), C.c_int, C.c_int, _P(Csr), _P(C.c_int), _P(C.c_int64)]
    ref.ref_summa.argtypes = [C.c_int, _P(Coo), _P(Coo), C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_uint64,
                              _P(Coo), _P(C.c_uint64), _P(C.c_double)]
    ref.ref_find_crossover_bundled.argtypes = [C.c_int, C.c_uint64, C.c_uint64, _P(C.c_uint64)]
    ref.ref_find_crossover_file.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.c_uint64, _P(C.c_uint64)]
    ref.ref_bundled_host_total.restype = C.c_double
    ref.ref_bundled_host_total.argtypes = [C.c_uint64, C.c_int]
    ref.ref_bundled_device_total.restype = C.c_double
    ref.ref_bundled_device_total.argtypes = [C.c_uint64, C.c_int]
    ref.ref_esc_rows_mt.argtypes = [C.c_int, _P(Csr), _P(Csr), C.c_int64, C.c_int64, C.c_int, _P(C.c_double),
                                    _P(C.c_int64), _P(C.c_int64), _P(C.c_uint64)]


class Mat:
    """Plain CSR/CSC triple with logical dims (ptr over rows, or cols if csc)."""

    def __init__(self, sr, nrows, ncols, ptr, idx, vals, csc=False):
        self.sr, self.nrows, self.ncols, self.csc = int(sr), int(nrows), int(ncols), csc
        self.ptr = np.ascontiguousarray(ptr, dtype=np.int64)
        self.idx = np.ascontiguousarray(idx, dtype=np.int64)
        self.vals = np.ascontiguousarray(np.asarray(vals).astype(_DT[self.sr], copy=False))

    @property
    def nnz(self):
        return int(self.idx.shape[0])

    def c(self):
        self._keep = (self.ptr, self.idx, self.vals)
        return Csr(self.nrows, self.ncols, self.nnz, self.ptr.ctypes.data_as(_P(C.c_int64)),
                   self.idx.ctypes.data_as(_P(C.c_int64)), self.vals.ctypes.data_as(C.c_void_p))

    @classmethod
    def of(cls, m):
        """From a product formats.CsrMatrix / CscMatrix."""
        if hasattr(m, "rowptr"):
            return cls(m.sr, m.nrows, m.ncols, m.rowptr, m.colids, m.values)
        return cls(m.sr, m.nrows, m.ncols, m.colptr, m.rowids, m.values, csc=True)


def _copy_out(ptr, n, dt):
    if n == 0 or not ptr:
        return np.zeros(0, dtype=dt)
    raw = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(n * dt.itemsize,))
    return raw.copy().view(dt)


def _take_csr(sr, c: Csr, csc=False, free=None):
    nseg = c.ncols if csc else c.nrows
    n = int(c.nnz)
    ptr = np.ctypeslib.as_array(c.ptr, shape=(nseg + 1,)).copy()
    idx = np.ctypeslib.as_array(c.idx, shape=(max(n, 1),))[:n].copy()
    dt = _DT[sr]
    vals = _copy_out(c.vals, n, dt)
    for p in (c.ptr, c.idx):
        free(C.cast(p, C.c_void_p))
    free(c.vals)
    return Mat(sr, c.nrows, c.ncols, ptr, idx, vals, csc)


def _take_coo(sr, c: Coo):
    n = int(c.nnz)
    r = np.ctypeslib.as_array(c.rows, shape=(max(n, 1),))[:n].copy()
    cc = np.ctypeslib.as_array(c.cols, shape=(max(n, 1),))[:n].copy()
    dt = _DT[sr]
    v = _copy_out(c.vals, n, dt)
    ref.ref_free(C.cast(c.rows, C.c_void_p))
    ref.ref_free(C.cast(c.cols, C.c_void_p))
    ref.ref_free(c.vals)
    return c.nrows, c.ncols, r, cc, v


def _coo_struct(nrows, ncols, rows, cols, vals, sr):
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    vals = np.ascontiguousarray(np.asarray(vals).astype(_DT[sr], copy=False))
    s = Coo(nrows, ncols, rows.shape[0], rows.ctypes.data_as(_P(C.c_int64)), cols.ctypes.data_as(_P(C.c_int64)),
            vals.ctypes.data_as(C.c_void_p))
    s._keep = (rows, cols, vals)
    return s


# ----------------------------------------------------------------- oracle
def orc_multiply(a: Mat, b: Mat, nthreads=0) -> Mat:
    out = Csr()
    rc = orc.orc_multiply(a.sr, C.byref(a.c()), C.byref(b.c()), nthreads, C.byref(out))
    assert rc == 0, "oracle multiply failed"
    return _take_csr(a.sr, out, free=orc.orc_free)


def orc_stream(a: Mat, b: Mat, lo=0, hi=None, nthreads=0, rownnz=False):
    hi = a.nrows if hi is None else hi
    s, z, f = C.c_uint64(), C.c_int64(), C.c_int64()
    rn = np.zeros(max(hi - lo, 1), dtype=np.int64) if rownnz else None
    rc = orc.orc_multiply_stream(a.sr, C.byref(a.c()), C.byref(b.c()), lo, hi, nthreads, C.byref(s),
                                 rn.ctypes.data_as(_P(C.c_int64)) if rownnz else None, C.byref(z), C.byref(f))
    assert rc == 0
    return int(s.value), int(z.value), int(f.value), (rn[: hi - lo] if rownnz else None)


def orc_checksum(m: Mat) -> int:
    out = C.c_uint64()
    assert orc.orc_checksum(m.sr, C.byref(m.c()), int(m.csc), C.byref(out)) == 0
    return int(out.value)


def orc_seed(nrows, ncols) -> int:
    return int(orc.orc_checksum_seed(nrows, ncols))


# -------------------------------------------------------------- reference
def _ok(rc):
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {ref.ref_last_error().decode()}")


def ref_generate_rmat(sr, scale, ef, seed):
    out = Coo()
    _ok(ref.ref_generate_rmat(sr, scale, ef, seed, C.byref(out)))
    return _take_coo(sr, out)


def ref_read_matrix_market(sr, path):
    """(status, message, (nrows, ncols, rows, cols, vals) or None)."""
    out = Coo()
    rc = ref.ref_read_matrix_market(sr, os.fsencode(path), C.byref(out))
    if rc != 0:
        return rc, ref.ref_last_error().decode(), None
    return 0, "", _take_coo(sr, out)


def ref_random_coo(sr, seed, nrows, ncols, density, exact=True):
    out = Coo()
    _ok(ref.ref_random_coo(sr, seed, nrows, ncols, density, int(exact), C.byref(out)))
    return _take_coo(sr, out)


def ref_esc(a: Mat, b: Mat, chunk=4096) -> Mat:
    out = Csr()
    _ok(ref.ref_esc_multiply(a.sr, C.byref(a.c()), C.byref(b.c()), chunk, C.byref(out)))
    return _take_csr(a.sr, out, free=ref.ref_free)


def ref_esc_status(a: Mat, b: Mat):
    out = Csr()
    return ref.ref_esc_multiply(a.sr, C.byref(a.c()), C.byref(b.c()), 4096, C.byref(out))


def ref_naive(a: Mat, b: Mat) -> Mat:
    out = Csr()
    _ok(ref.ref_naive_multiply(a.sr, C.byref(a.c()), C.byref(b.c()), C.byref(out)))
    return _take_csr(a.sr, out, free=ref.ref_free)


def ref_coo_to_csr(sr, nrows, ncols, rows, cols, vals) -> Mat:
    out = Csr()
    _ok(ref.ref_coo_to_csr(sr, C.byref(_coo_struct(nrows, ncols, rows, cols, vals, sr)), C.byref(out)))
    return _take_csr(sr, out, free=ref.ref_free)


def ref_coo_to_csc(sr, nrows, ncols, rows, cols, vals) -> Mat:
    out = Csr()
    _ok(ref.ref_coo_to_csc(sr, C.byref(_coo_struct(nrows, ncols, rows, cols, vals, sr)), C.byref(out)))
    return _take_csr(sr, out, csc=True, free=ref.ref_free)


def ref_distribute_block(sr, nrows, ncols, rows, cols, vals, p, rank):
    """The reference's distribute on a p-rank square grid: (block as CSC Mat,
    is_dcsc, (row_begin, row_end, col_begin, col_end))."""
    out = Csr()
    flag = C.c_int()
    ext = (C.c_int64 * 4)()
    _ok(ref.ref_distribute_block(sr, C.byref(_coo_struct(nrows, ncols, rows, cols, vals, sr)), p, rank,
                                 C.byref(out), C.byref(flag), ext))
    return _take_csr(sr, out, csc=True, free=ref.ref_free), bool(flag.value), tuple(ext)


def ref_checksum(m: Mat) -> int:
    out = C.c_uint64()
    fn = ref.ref_checksum_csc if m.csc else ref.ref_checksum_csr
    _ok(fn(m.sr, C.byref(m.c()), C.byref(out)))
    return int(out.value)


def ref_slice(m: Mat, by_rows, b, e) -> Mat:
    out = Csr()
    _ok(ref.ref_csr_slice(m.sr, C.byref(m.c()), int(by_rows), b, e, C.byref(out)))
    return _take_csr(m.sr, out, free=ref.ref_free)


def ref_merge(parts, stages, rounds, block_rows, block_cols) -> Mat:
    n = len(parts)
    arr = (Csr * n)(*[p.c() for p in parts])
    out = Csr()
    _ok(ref.ref_merge_partials(parts[0].sr, n, arr, (C.c_int * n)(*stages), (C.c_int * n)(*rounds),
                               block_rows, block_cols, C.byref(out)))
    return _take_csr(parts[0].sr, out, csc=True, free=ref.ref_free)


def ref_block_range(n, q, idx):
    b, e = C.c_int64(), C.c_int64()
    ref.ref_block_range(n, q, idx, C.byref(b), C.byref(e))
    return b.value, e.value


def ref_round_range(n, rounds, r):
    b, e = C.c_int64(), C.c_int64()
    ref.ref_round_range(n, rounds, r, C.byref(b), C.byref(e))
    return b.value, e.value


def ref_summa(sr, nrows, ncols, rows, cols, vals, p, two_round=True, mode=2, threshold=0, chunk=4096):
    a = _coo_struct(nrows, ncols, rows, cols, vals, sr)
    out = Coo()
    cs = C.c_uint64()
    led = (C.c_double * 12)()
    rc = ref.ref_summa(sr, C.byref(a), C.byref(a), p, int(two_round), mode, threshold, chunk, C.byref(out),
                       C.byref(cs), led)
    if rc != 0:
        return rc, ref.ref_last_error().decode(), None, None
    return 0, _take_coo(sr, out), int(cs.value), list(led)


def ref_find_crossover_file(path, fanout, lo, hi):
    """The reference's find_crossover on LatencyModel::load_file(path); None without a crossover."""
    out = C.c_uint64()
    rc = ref.ref_find_crossover_file(path.encode(), fanout, lo, hi, C.byref(out))
    assert rc >= 0, ref.ref_last_error()
    return int(out.value) if rc == 1 else None


def ref_find_crossover(fanout, lo, hi):
    out = C.c_uint64()
    return int(out.value) if ref.ref_find_crossover_bundled(fanout, lo, hi, C.byref(out)) else None


def ref_esc_rows_mt(a: Mat, b: Mat, lo, hi, nthreads):
    sec, nnz, fl, cs = C.c_double(), C.c_int64(), C.c_int64(), C.c_uint64()
    _ok(ref.ref_esc_rows_mt(a.sr, C.byref(a.c()), C.byref(b.c()), lo, hi, nthreads, C.byref(sec), C.byref(nnz),
                            C.byref(fl), C.byref(cs)))
    return sec.value, nnz.value, fl.value, int(cs.value)
