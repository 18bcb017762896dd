"""GPU parity of the bitmap-rank local multiply (csrc/bitmap_rank.cuh): long
rows (F > 2048 products) go through a symbolic bitmap pass, exact row
pointers and a rank-space fold written straight into C.  Every case is
checked against the CPU oracle (and, for the headline configuration, the
oracle's streaming restatement at full size), through the C-ABI."""
import os

import numpy as np
import pytest

import oracle_bind as ob
from helpers import RTOL, assert_same, to_mat
from paper_2504_06408_b200 import DeviceCsr, esc_multiply, generators, local_multiply
from paper_2504_06408_b200._lib import lib
from paper_2504_06408_b200.formats import CsrMatrix, coo_to_csr

pytestmark = pytest.mark.gpu

BIN_BITMAP = 10
MODE_BITMAP = 3
MODE_PATTERN = 4


def _exact(sr, rng, n):
    from golden.make_golden import exact_values
    return exact_values(sr, rng, n)


def _wide_case(sr, rng, ncols, nb, blen, row_segs):
    b_cols = [np.sort(rng.choice(ncols, blen, replace=False)) for _ in range(nb)]
    bptr = np.concatenate([[0], np.cumsum([len(x) for x in b_cols])]).astype(np.int64)
    bc = np.concatenate(b_cols).astype(np.int64)
    b = CsrMatrix(sr, nb, ncols, bptr, bc, _exact(sr, rng, bc.size))
    rows = [np.sort(rng.choice(nb, k, replace=False)) for k in row_segs]
    aptr = np.concatenate([[0], np.cumsum([len(x) for x in rows])]).astype(np.int64)
    ac = np.concatenate(rows).astype(np.int64)
    a = CsrMatrix(sr, len(rows), nb, aptr, ac, _exact(sr, rng, ac.size))
    return a, b


@pytest.mark.parametrize("sr", [0, 1, 2, 3, 4, 5])
def test_rank_windows_against_oracle(ctx, sr):
    """Rows from 1 to ~190K outputs over a 200K-column C: single-window rows
    and rows folded in several rank windows (window = 8K..64K outputs by value
    width), mixed with short rows on the hash / ESC bins."""
    rng = np.random.default_rng(40 + sr)
    a, b = _wide_case(sr, rng, 200_000, 96, 3000, [1, 2, 3, 5, 8, 14, 30, 60, 96, 0, 1])
    # a few short rows (hash / ESC bins) next to the long ones
    st = {}
    got = esc_multiply(a, b, ctx=ctx, stats=st)
    want = ob.orc_multiply(to_mat(a), to_mat(b))
    assert_same(got, want, sr, rtol=RTOL if sr == 0 else None)
    assert st["output_mode"] == (MODE_PATTERN if sr == 2 else MODE_BITMAP)
    lens = np.diff(b.rowptr)
    long_rows = sum(int(lens[a.colids[a.rowptr[i]:a.rowptr[i + 1]]].sum()) > 2048 for i in range(a.nrows))
    assert st["rows_per_bin"][BIN_BITMAP] == long_rows, st["rows_per_bin"]
    assert got.nnz > 3 * 65536  # windows exercised for every value width


@pytest.mark.parametrize("sr", [0, 2, 4, 5])
def test_same_as_bins_pipeline_on_rmat(ctx, sr):
    """R-MAT scale 13: the bitmap-rank pipeline and the per-bin pipeline give
    the same C."""
    m = coo_to_csr(generators.generate_rmat(sr, 13, 16.0, 7))
    d = DeviceCsr.upload(ctx, m)
    st = {}
    got = local_multiply(d, d, stats=st).download()
    assert st["output_mode"] == (MODE_PATTERN if sr == 2 else MODE_BITMAP) and st["rows_per_bin"][BIN_BITMAP] > 0
    ctx.set_pipeline(ctx.PIPE_BINS)
    try:
        st2 = {}
        want = local_multiply(d, d, stats=st2).download()
    finally:
        ctx.set_pipeline(ctx.PIPE_AUTO)
    assert st2["output_mode"] not in (MODE_BITMAP, MODE_PATTERN)
    assert_same(got, want, sr, rtol=RTOL if sr == 0 else None)
    assert_same(got, ob.orc_multiply(to_mat(m), to_mat(m)), sr, rtol=RTOL if sr == 0 else None)


def test_zero_products_are_dropped(ctx):
    """Tropical (min, saturating +): products that saturate to INT32_MAX are
    the semiring zero; the symbolic pass marked their columns, so the
    zero-valued entries are compacted away (local_spgemm.hpp:57-58)."""
    rng = np.random.default_rng(11)
    ncols, nb = 100_000, 8
    bptr = np.arange(0, 1000 * nb + 1, 1000, dtype=np.int64)
    bcols = np.concatenate([np.sort(rng.choice(ncols, 1000, replace=False)) for _ in range(nb)]).astype(np.int64)
    big = (1 << 30) + 5
    bvals = rng.integers(1, 100, bcols.size).astype(np.int32)
    bvals[:2000] = big
    b = CsrMatrix(4, nb, ncols, bptr, bcols, bvals)
    avals = np.full(nb, 3, dtype=np.int32)
    avals[:2] = big
    a = CsrMatrix(4, 1, nb, np.array([0, nb], dtype=np.int64), np.arange(nb, dtype=np.int64), avals)
    st = {}
    got = esc_multiply(a, b, ctx=ctx, stats=st)
    assert_same(got, ob.orc_multiply(to_mat(a), to_mat(b)), 4)
    assert st["rows_per_bin"][BIN_BITMAP] == 1


def test_fp64_exact_cancellation_is_dropped(ctx):
    """(+, x) over fp64: a row whose products cancel to exactly 0.0 in some
    columns (B rows k and k+20 identical, A weights +1 / -1) loses those
    entries, as the reference's fold-then-drop does."""
    rng = np.random.default_rng(5)
    ncols, half, blen = 50_000, 20, 120
    base_cols = [np.sort(rng.choice(ncols, blen, replace=False)) for _ in range(half)]
    base_vals = [rng.integers(1, 9, blen).astype(np.float64) for _ in range(half)]
    cols = base_cols + base_cols + [np.sort(rng.choice(ncols, blen, replace=False))]
    vals = base_vals + base_vals + [rng.integers(1, 9, blen).astype(np.float64)]
    bptr = np.concatenate([[0], np.cumsum([len(x) for x in cols])]).astype(np.int64)
    b = CsrMatrix(0, 2 * half + 1, ncols, bptr, np.concatenate(cols).astype(np.int64), np.concatenate(vals))
    ac = np.arange(2 * half + 1, dtype=np.int64)
    av = np.concatenate([np.ones(half), -np.ones(half), [2.0]])
    a = CsrMatrix(0, 1, 2 * half + 1, np.array([0, ac.size], dtype=np.int64), ac, av)
    st = {}
    got = esc_multiply(a, b, ctx=ctx, stats=st)
    want = ob.orc_multiply(to_mat(a), to_mat(b))
    assert_same(got, want, 0, rtol=RTOL)
    assert st["rows_per_bin"][BIN_BITMAP] == 1
    assert got.nnz < 2 * half * blen  # the cancelled columns are gone


def test_headline_config2_full_size_against_streaming_oracle(ctx):
    """BASELINE config 2 exactly as bench.py runs it (R-MAT scale 18, edge
    factor 16, vertices relabelled by the seeded permutation, (min, +) int32):
    C = A.A through local_multiply on one GPU, compared with the oracle's
    streaming restatement over all host cores — order-free checksum, nnz(C),
    the product count and every row's nnz."""
    coo = generators.generate_rmat(4, 18, 16.0, 1)
    coo = generators.permute_symmetric(coo, 1)
    a = generators.coo_to_csr_fast(coo)
    d = DeviceCsr.upload(ctx, a)
    st = {}
    c = local_multiply(d, d, stats=st)
    assert st["products"] == 2934326978 and c.nnz == 1281547801
    csum = c.checksum()
    rownnz = np.diff(c.rowptr_host())
    del c
    s, z, f, rn = ob.orc_stream(to_mat(a), to_mat(a), rownnz=True, nthreads=min(64, os.cpu_count() or 8))
    assert (z, f) == (1281547801, 2934326978)
    assert np.array_equal(rownnz, rn)
    assert csum == (ob.orc_seed(a.nrows, a.ncols) + s) % (1 << 64)


@pytest.mark.parametrize("ncols", [3000, 200_000, 1_500_000])
def test_boolean_pattern_path_any_width(ctx, ncols):
    """Boolean (pattern-only): long rows take two column-only passes over
    column super-panels of <= 2^19 columns (count, then emit straight into C
    with every value one()) at any output width — 1.5M columns means three
    super-panels per row.  An explicit false in an operand sends the call
    down the general pipeline (its products must vanish)."""
    rng = np.random.default_rng(17)
    nb = 60
    lens = rng.integers(200, min(ncols // 2, 4000), nb)
    bptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    bcols = np.concatenate([np.sort(rng.choice(ncols, L, replace=False)) for L in lens]).astype(np.int64)
    b = CsrMatrix(2, nb, ncols, bptr, bcols, np.ones(bcols.size, np.uint8))
    rows = [np.sort(rng.choice(nb, k, replace=False)) for k in (1, 4, 12, 30, 60, 0, 2)]
    aptr = np.concatenate([[0], np.cumsum([len(x) for x in rows])]).astype(np.int64)
    acols = np.concatenate(rows).astype(np.int64)
    a = CsrMatrix(2, len(rows), nb, aptr, acols, np.ones(acols.size, np.uint8))
    st = {}
    got = esc_multiply(a, b, ctx=ctx, stats=st)
    assert_same(got, ob.orc_multiply(to_mat(a), to_mat(b)), 2)
    assert st["output_mode"] == MODE_PATTERN and st["rows_per_bin"][BIN_BITMAP] >= 3, st
    bz = CsrMatrix(2, nb, ncols, bptr, bcols, np.ones(bcols.size, np.uint8))
    bz.values[::7] = 0  # explicit false entries
    st2 = {}
    got2 = esc_multiply(a, bz, ctx=ctx, stats=st2)
    assert_same(got2, ob.orc_multiply(to_mat(a), to_mat(bz)), 2)
    assert st2["output_mode"] != MODE_PATTERN
