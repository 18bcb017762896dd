"""GPU distribute (spg_distribute, csrc/distribute.cu) against the reference's
own distribute (dist_matrix.hpp:69-111) and coo_to_csc (formats.hpp:138-180),
compiled from its headers (oracle/_ref): every block's CSC pattern, values,
DCSC choice and extents, bit-exact — including duplicate tuples in random
order (folded with SR::add in input order, so even fp64 sums match bit for
bit), explicit zeros and cancellations (dropped), and non-square grids."""
import numpy as np
import pytest

import oracle_bind as ob
from helpers import assert_same
from paper_2504_06408_b200 import errors, generators
from paper_2504_06408_b200.formats import CooMatrix, dcsc_decompress
from paper_2504_06408_b200.summa import block_range, distribute, local_block

pytestmark = pytest.mark.gpu


def _csc_of(blk):
    s = blk.storage
    return dcsc_decompress(s) if blk.is_dcsc else s


def _values(sr, rng, n):
    if sr == 0:
        return rng.standard_normal(n)  # non-integer: any reordering of the fold would show
    if sr == 1:
        return rng.integers(1, 50, n).astype(np.float64)
    if sr == 2:
        return (rng.random(n) < 0.9).astype(np.uint8)  # explicit false entries
    if sr == 3:
        v = np.zeros(n, dtype=ob._DT[3])
        v["weight"] = rng.integers(1, 6, n)  # ties: the fold order picks the payload
        v["payload"] = rng.integers(0, 1000, n)
        return v
    if sr == 4:
        v = rng.integers(0, 100, n).astype(np.int32)
        v[rng.random(n) < 0.05] = np.iinfo(np.int32).max  # the semiring zero
        return v
    v = np.zeros(n, dtype=ob._DT[5])
    v["w"] = rng.integers(0, 8, n) / 4.0  # ties and zeros
    v["tag"] = rng.integers(0, 1 << 62, n, dtype=np.uint64)
    return v


def _messy_coo(sr, rng, nrows, ncols, n):
    """Random order, ~30 % duplicates, explicit zeros and exact cancellations."""
    r = rng.integers(0, nrows, n)
    c = rng.integers(0, ncols, n)
    dup = rng.random(n) < 0.3
    src = rng.integers(0, n, n)
    r[dup], c[dup] = r[src[dup]], c[src[dup]]
    v = _values(sr, rng, n)
    if sr == 0:
        v[rng.random(n) < 0.03] = 0.0
        k = np.nonzero(dup)[0][:50]  # x then -x at the same coordinate: cancels to exactly 0
        v[k] = -v[src[k]]
    return CooMatrix(sr, nrows, ncols, r, c, v)


@pytest.mark.parametrize("sr", [0, 1, 2, 3, 4, 5])
@pytest.mark.parametrize("p", [1, 4, 9])
def test_blocks_match_reference_distribute(ctx, sr, p):
    rng = np.random.default_rng(100 * sr + p)
    m = _messy_coo(sr, rng, 301, 257, 6000)
    blocks = distribute(ctx, m, int(np.sqrt(p)), int(np.sqrt(p)))
    for rank, blk in enumerate(blocks):
        want, want_dcsc, ext = ob.ref_distribute_block(sr, m.nrows, m.ncols, m.rows, m.cols, m.values, p, rank)
        assert (blk.rows + blk.cols) == ext
        assert blk.is_dcsc == want_dcsc
        assert_same(_csc_of(blk), want, sr)


@pytest.mark.parametrize("sr", [0, 4])
@pytest.mark.parametrize("grid", [(1, 2), (2, 4), (3, 1), (1, 5)])
def test_rectangular_grids_match_reference_coo_to_csc(ctx, sr, grid):
    """pr x pc grids (the reference's distribute is square-only): each block
    equals the reference's coo_to_csc of the tuples it owns, in input order."""
    pr, pc = grid
    rng = np.random.default_rng(7 + pr * 10 + pc)
    m = _messy_coo(sr, rng, 203, 350, 5000)
    blocks = distribute(ctx, m, pr, pc)
    for rank, blk in enumerate(blocks):
        rb, re = block_range(m.nrows, pr, rank // pc)
        cb, ce = block_range(m.ncols, pc, rank % pc)
        sel = (m.rows >= rb) & (m.rows < re) & (m.cols >= cb) & (m.cols < ce)
        want = ob.ref_coo_to_csc(sr, re - rb, ce - cb, m.rows[sel] - rb, m.cols[sel] - cb, m.values[sel])
        assert blk.rows == (rb, re) and blk.cols == (cb, ce)
        assert blk.is_dcsc == (2 * int(np.count_nonzero(np.diff(want.ptr))) < ce - cb)
        assert_same(_csc_of(blk), want, sr)
        one = distribute(ctx, m, pr, pc, only_rank=rank)  # one process per GPU builds only its own
        assert one.rows == blk.rows and one.is_dcsc == blk.is_dcsc
        assert_same(_csc_of(one), want, sr)


def test_rmat_blocks_equal_host_local_block(ctx):
    """Normalised R-MAT (the bench inputs): the GPU blocks equal the host
    restatement summa.local_block, DCSC choice included."""
    m = generators.generate_rmat(4, 12, 16.0, 3)
    for pr, pc in [(1, 1), (2, 2), (2, 4)]:
        blocks = distribute(ctx, m, pr, pc)
        for rank, blk in enumerate(blocks):
            host = local_block(m, pr, pc, rank // pc, rank % pc)
            assert blk.is_dcsc == host.is_dcsc and blk.rows == host.rows and blk.cols == host.cols
            assert_same(_csc_of(blk), _csc_of(host), 4)


def test_hypersparse_blocks_are_dcsc_and_empty_input(ctx):
    m = CooMatrix(4, 1000, 4000, np.array([5, 700, 5]), np.array([10, 3999, 2100]),
                  np.array([1, 2, 3], dtype=np.int32))
    blocks = distribute(ctx, m, 2, 2)
    assert all(b.is_dcsc for b in blocks)
    assert [b.storage.jc.tolist() for b in blocks] == [[10], [100], [], [1999]]
    empty = CooMatrix(4, 10, 6, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int32))
    for b in distribute(ctx, empty, 2, 3):
        assert b.is_dcsc and b.storage.nnz == 0 and b.storage.cp.tolist() == [0]


def test_tuple_outside_matrix_is_malformed(ctx):
    m = CooMatrix(4, 10, 10, np.array([1, 10]), np.array([1, 2]), np.array([1, 2], dtype=np.int32))
    with pytest.raises(errors.MalformedInputError):
        distribute(ctx, m, 1, 2)
    with pytest.raises(errors.GridError):
        distribute(ctx, m, 2, 2, only_rank=4)
