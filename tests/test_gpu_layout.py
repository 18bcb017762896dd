"""GPU parity of the SUMMA layout operators against reference-generated
fixtures (tests/golden/make_golden.py) and the reference library:

  csr_row_slice / csr_col_slice   summa.hpp:57-98   -> spg_csr_slice
  prepare_block (DCSC branch)     summa.hpp:30-53 + dcsc_decompress,
                                  formats.hpp:220-250 -> spg_prepare_block
"""
import ctypes as C

import numpy as np
import pytest

import oracle_bind as ob
from helpers import assert_same, unpack
from paper_2504_06408_b200 import DeviceCsr
from paper_2504_06408_b200._lib import DCsr, HDcsc, check, lib
from paper_2504_06408_b200.formats import CscMatrix, CsrMatrix

pytestmark = pytest.mark.gpu


def _slice(ctx, m, by_rows, b, e):
    d = DeviceCsr.upload(ctx, m)
    out = DCsr()
    check(lib.spg_csr_slice(ctx.handle, int(m.sr), C.byref(d.d), int(by_rows), int(b), int(e), C.byref(out)),
          ctx.handle)
    return DeviceCsr(ctx, m.sr, out).download()


def test_row_and_col_slices_match_reference_fixtures(golden, ctx):
    m = unpack(golden, "slice_m", 4)
    assert_same(_slice(ctx, m, True, 7, 31), unpack(golden, "slice_rows", 4), 4)
    assert_same(_slice(ctx, m, False, 13, 52), unpack(golden, "slice_cols", 4), 4)


@pytest.mark.parametrize("sr", [0, 1, 2, 4, 5])
def test_slices_random_against_reference(ctx, sr):
    from golden.make_golden import random_csr
    rng = np.random.default_rng(17 + sr)
    m = random_csr(sr, rng, 200, 300, 0.05)
    for b, e in [(0, 0), (0, 200), (37, 38), (150, 200)]:
        assert_same(_slice(ctx, CsrMatrix(sr, 200, 300, m.ptr, m.idx, m.vals), True, b, e),
                    ob.ref_slice(m, True, b, e), sr)
    for b, e in [(0, 0), (0, 300), (5, 6), (120, 299)]:
        assert_same(_slice(ctx, CsrMatrix(sr, 200, 300, m.ptr, m.idx, m.vals), False, b, e),
                    ob.ref_slice(m, False, b, e), sr)


def _dcsc_of(csc):
    lens = np.diff(csc.ptr)
    jc = np.nonzero(lens)[0].astype(np.int64)
    cp = np.concatenate([[0], np.cumsum(lens[jc])]).astype(np.int64)
    return jc, cp


@pytest.mark.parametrize("sr", [0, 1, 2, 4, 5])
def test_dcsc_prepare_matches_reference_decompress(ctx, sr):
    """A hypersparse block (most columns empty) given as DCSC: the device
    decompress + transpose reinterpretation equals the reference's
    dcsc_decompress(csc_to_dcsc(block)) read as the CSR of the transpose."""
    from golden.make_golden import random_csr
    rng = np.random.default_rng(5 + sr)
    nrows, ncols = 90, 400
    m = random_csr(sr, rng, ncols, nrows, 0.004)  # CSR of B^T == CSC of the block B (nrows x ncols)
    csc = ob.Mat(sr, nrows, ncols, m.ptr, m.idx, m.vals, csc=True)
    jc_len = C.c_int64()
    out = ob.Csr()
    assert ob.ref.ref_dcsc_roundtrip(sr, C.byref(csc.c()), C.byref(jc_len), C.byref(out)) == 0
    want = ob._take_csr(sr, out, csc=True, free=ob.ref.ref_free)
    jc, cp = _dcsc_of(csc)
    assert jc.size == jc_len.value and 2 * jc.size < ncols  # the DCSC choice (dist_matrix.hpp:97-108)
    ri = np.ascontiguousarray(csc.idx, dtype=np.int64)
    v = np.ascontiguousarray(csc.vals)
    h = HDcsc(nrows, ncols, ri.shape[0], jc.shape[0], jc.ctypes.data_as(C.POINTER(C.c_int64)),
              cp.ctypes.data_as(C.POINTER(C.c_int64)), ri.ctypes.data_as(C.POINTER(C.c_int64)),
              v.ctypes.data_as(C.c_void_p))
    d = DCsr()
    check(lib.spg_prepare_block(ctx.handle, sr, None, C.byref(h), C.byref(d)), ctx.handle)
    got = DeviceCsr(ctx, sr, d).download()  # CSR of the transpose: rows = block columns
    assert got.nrows == ncols and got.ncols == nrows
    assert np.array_equal(got.rowptr, want.ptr) and np.array_equal(got.colids, want.idx)
    assert got.values.tobytes() == want.vals.tobytes()


def test_dcsc_prepare_rejects_malformed(ctx):
    from paper_2504_06408_b200 import errors
    jc = np.array([3, 2], dtype=np.int64)  # not increasing
    cp = np.array([0, 1, 2], dtype=np.int64)
    ri = np.array([0, 1], dtype=np.int64)
    v = np.array([1, 2], dtype=np.int32)
    h = HDcsc(4, 5, 2, 2, jc.ctypes.data_as(C.POINTER(C.c_int64)), cp.ctypes.data_as(C.POINTER(C.c_int64)),
              ri.ctypes.data_as(C.POINTER(C.c_int64)), v.ctypes.data_as(C.c_void_p))
    d = DCsr()
    with pytest.raises(errors.MalformedInputError):
        check(lib.spg_prepare_block(ctx.handle, 4, None, C.byref(h), C.byref(d)), ctx.handle)
    h0 = HDcsc(4, 5, 0, 0, None, None, None, None)  # njc == 0 still needs cp[1]
    with pytest.raises(errors.MalformedInputError):
        check(lib.spg_prepare_block(ctx.handle, 4, None, C.byref(h0), C.byref(d)), ctx.handle)
