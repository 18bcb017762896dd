"""A user-defined semiring plugged in from OUTSIDE the library (the
reference's SemiringLike plug-in model, semiring.hpp:28-40): the (max, min)
bottleneck semiring over int32, compiled from tests/custom_sr/maxmin_sr.cu
into its own shared library with SPG_INSTANTIATE and registered at run time
(spg_register_semiring).  GPU results are checked against a dense numpy
(max, min) product — exact integer arithmetic."""
import os

import numpy as np
import pytest

from paper_2504_06408_b200 import DeviceCsr, errors, esc_multiply, local_multiply, matrix_checksum, register_semiring
from paper_2504_06408_b200._lib import lib
from paper_2504_06408_b200.formats import CsrMatrix

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "tests", "custom_sr", "libmaxmin_sr.so")
NEG = np.iinfo(np.int32).min


@pytest.fixture(scope="module")
def maxmin():
    if not os.path.exists(SO):
        pytest.fail("tests/custom_sr/libmaxmin_sr.so missing: run `make custom_sr` (part of `make all`)")
    return register_semiring(SO, "spg_user_maxmin_i32_ops", "int32")


def test_registration(maxmin):
    assert maxmin >= 6
    assert lib.spg_semiring_name(maxmin).decode() == "maxmin_i32"
    assert lib.spg_semiring_by_name(b"maxmin_i32") == maxmin
    assert lib.spg_value_size(maxmin) == 4
    assert lib.spg_semiring_is_commutative(maxmin) == 1
    # the same table again: same id
    assert register_semiring(SO, "spg_user_maxmin_i32_ops", "int32") == maxmin
    with pytest.raises(errors.ShapeError):  # dtype must match value_type's size
        register_semiring(SO, "spg_user_maxmin_i32_ops", "int64")


def _rand_csr(sr, rng, m, k, dens):
    mask = rng.random((m, k)) < dens
    r, c = np.nonzero(mask)
    vals = rng.integers(1, 1000, r.size).astype(np.int32)
    ptr = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=m))]).astype(np.int64)
    return CsrMatrix(sr, m, k, ptr, c.astype(np.int64), vals)


def _dense(m):
    d = np.full((m.nrows, m.ncols), NEG, dtype=np.int64)
    rows = np.repeat(np.arange(m.nrows), np.diff(m.rowptr))
    d[rows, m.colids] = m.values
    return d


def _maxmin(a, b):
    out = np.full((a.shape[0], b.shape[1]), NEG, dtype=np.int64)
    for k in range(a.shape[1]):
        out = np.maximum(out, np.minimum(a[:, k:k + 1], b[k:k + 1, :]))
    return out


def _check(got, a, b):
    want = _maxmin(_dense(a), _dense(b))
    rows, cols = np.nonzero(want != NEG)
    assert np.array_equal(np.diff(got.rowptr), np.bincount(rows, minlength=a.nrows))
    assert np.array_equal(got.colids, cols)
    assert np.array_equal(got.values, want[rows, cols].astype(np.int32))


@pytest.mark.gpu
@pytest.mark.parametrize("pipeline", [0, 1])
def test_custom_semiring_multiply_against_dense(ctx, maxmin, pipeline):
    """Short rows (ESC / hash bins) and long rows (> 2048 products: the
    bitmap-rank kernels, or dense panels / bit-rank with the per-bin
    pipeline), all instantiated in the user's library."""
    rng = np.random.default_rng(3)
    a = _rand_csr(maxmin, rng, 60, 1500, 0.02)
    a2 = _rand_csr(maxmin, rng, 6, 1500, 0.6)  # long rows
    a = CsrMatrix(maxmin, 66, 1500, np.concatenate([a.rowptr, a.rowptr[-1] + a2.rowptr[1:]]),
                  np.concatenate([a.colids, a2.colids]), np.concatenate([a.values, a2.values]))
    b = _rand_csr(maxmin, rng, 1500, 2500, 0.02)
    ctx.set_pipeline(pipeline)
    try:
        st = {}
        got = esc_multiply(a, b, ctx=ctx, stats=st)
    finally:
        ctx.set_pipeline(0)
    _check(got, a, b)
    if pipeline == 0:
        assert st["rows_per_bin"][10] >= 6 and st["output_mode"] == 3


@pytest.mark.gpu
def test_custom_semiring_device_path_and_checksum(ctx, maxmin):
    rng = np.random.default_rng(4)
    a = _rand_csr(maxmin, rng, 300, 300, 0.03)
    d = DeviceCsr.upload(ctx, a)
    c = local_multiply(d, d)
    got = c.download()
    _check(got, a, a)
    assert c.checksum() == matrix_checksum(got, ctx=ctx)


@pytest.mark.gpu
def test_custom_semiring_distribute_folds_duplicates(ctx, maxmin):
    """spg_distribute with the user's semiring: duplicate tuples fold with the
    user's add (max) through the fold_runs entry of its ops table, and the
    (max, min) zero (INT32_MIN) is dropped."""
    from paper_2504_06408_b200.formats import CooMatrix, dcsc_decompress
    from paper_2504_06408_b200.summa import distribute
    rng = np.random.default_rng(9)
    n, nnz = 120, 3000
    r = rng.integers(0, n, nnz)
    c = rng.integers(0, n, nnz)
    v = rng.integers(-50, 1000, nnz).astype(np.int32)
    v[rng.random(nnz) < 0.05] = NEG
    m = CooMatrix(maxmin, n, n, r, c, v)
    want = np.full((n, n), NEG, dtype=np.int64)
    np.maximum.at(want, (r, c), v.astype(np.int64))
    for blk in distribute(ctx, m, 2, 2):
        s = dcsc_decompress(blk.storage) if blk.is_dcsc else blk.storage
        (rb, re), (cb, ce) = blk.rows, blk.cols
        d = np.full((re - rb, ce - cb), NEG, dtype=np.int64)
        cols = np.repeat(np.arange(ce - cb), np.diff(s.colptr))
        d[s.rowids, cols] = s.values
        assert np.array_equal(d, want[rb:re, cb:ce])
        assert not np.any(s.values == NEG)
