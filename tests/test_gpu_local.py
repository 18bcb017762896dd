"""GPU parity: the sm_100a local multiply / merge / checksum against the
reference (golden fixtures) and the CPU oracle, through the C-ABI."""
import numpy as np
import pytest

import oracle_bind as ob
from helpers import RTOL, assert_same, ptr_idx_vals, to_mat, unpack
from paper_2504_06408_b200 import (DeviceCsr, errors, esc_multiply, generators, local_multiply,
                                   matrix_checksum, merge_partials)
from paper_2504_06408_b200._lib import lib
from paper_2504_06408_b200.formats import CscMatrix, CsrMatrix, coo_to_csr

pytestmark = pytest.mark.gpu


def test_all_golden_local_cases_bit_exact(golden, ctx):
    for key in golden["mul_cases"]:
        sr = int(str(key).split("_")[1])
        a, b = unpack(golden, key + "_a", sr), unpack(golden, key + "_b", sr)
        want = unpack(golden, key + "_c", sr)
        st = {}
        got = esc_multiply(a, b, ctx=ctx, stats=st)
        assert_same(got, want, sr)  # integer-valued draws: bit-exact for every semiring
        assert matrix_checksum(got, ctx=ctx) == int(golden[key + "_csum"][0])
        assert st["kernels"] > 0


def test_spec_examples(golden, ctx):
    a = CsrMatrix(0, 2, 2, np.array([0, 2, 3]), np.array([0, 1, 1]), np.array([1.0, 2.0, 3.0]))
    got = esc_multiply(a, a, ctx=ctx)
    assert got.values.tolist() == [1.0, 8.0, 9.0]
    assert_same(got, unpack(golden, "spec_aa", 0), 0)
    w = CsrMatrix(1, 3, 3, np.array([0, 2, 4, 5]), np.array([0, 1, 1, 2, 2]), np.array([0.0, 1.0, 0.0, 2.0, 0.0]))
    assert_same(esc_multiply(w, w, ctx=ctx), unpack(golden, "spec_ww", 1), 1)


def test_config1_er4096_fp64_within_tolerance(golden, ctx):
    r, c, v = golden["er4096_rows"], golden["er4096_cols"], golden["er4096_vals"]
    from paper_2504_06408_b200.formats import CooMatrix
    a = coo_to_csr(CooMatrix(0, 4096, 4096, r, c, v))
    got = esc_multiply(a, a, ctx=ctx)
    assert_same(got, unpack(golden, "er4096_c", 0), 0, rtol=RTOL)


def test_shape_error(ctx):
    a = CsrMatrix(0, 2, 3, np.array([0, 0, 0]), np.zeros(0, np.int64), np.zeros(0))
    b = CsrMatrix(0, 2, 2, np.array([0, 0, 0]), np.zeros(0, np.int64), np.zeros(0))
    with pytest.raises(errors.ShapeError):
        esc_multiply(a, b, ctx=ctx)


def test_empty_and_zero_sized(ctx):
    for (m, k, n) in [(0, 0, 0), (5, 0, 7), (0, 4, 3), (6, 6, 6)]:
        a = CsrMatrix(4, m, k, np.zeros(m + 1, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int32))
        b = CsrMatrix(4, k, n, np.zeros(k + 1, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int32))
        got = esc_multiply(a, b, ctx=ctx)
        assert got.nrows == m and got.ncols == n and got.nnz == 0 and got.rowptr.tolist() == [0] * (m + 1)


def _rand(sr, rng, m, k, dens):
    from golden.make_golden import exact_values
    mask = rng.random((m, k)) < dens
    r, c = np.nonzero(mask)
    vals = exact_values(sr, rng, r.size)
    ptr = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=m))]).astype(np.int64)
    return CsrMatrix(sr, m, k, ptr, c.astype(np.int64), vals)


@pytest.mark.parametrize("sr", [0, 1, 2, 3, 4, 5])
def test_every_bin_against_oracle(bins_ctx, sr):
    """Rows engineered to land in every accumulator bin: empty, <=32 products
    (warp-ESC), the four hash-table sizes and the dense global accumulator."""
    rng = np.random.default_rng(100 + sr)
    n = 40000
    # B: row k has (k % 97) + 1 entries spread over n columns (sorted, unique)
    lens = (np.arange(2000) % 97) + 1
    bptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    bcols = np.concatenate([np.sort(rng.choice(n, L, replace=False)) for L in lens]).astype(np.int64)
    from golden.make_golden import exact_values
    b = CsrMatrix(sr, 2000, n, bptr, bcols, exact_values(sr, rng, bcols.size))
    # A: rows with 0, 1, 3, 20, 120, 600, 1500 entries
    sizes = [0, 1, 3, 20, 120, 600, 1500, 0, 2, 60]
    rows = []
    for s in sizes:
        rows.append(np.sort(rng.choice(2000, s, replace=False)))
    rows[1] = np.array([5])       # 6 products  -> warp-ESC bin
    rows[8] = np.array([3, 200])  # 4 + 7 = 11 products -> warp-ESC bin
    aptr = np.concatenate([[0], np.cumsum([len(x) for x in rows])]).astype(np.int64)
    acols = np.concatenate(rows).astype(np.int64)
    a = CsrMatrix(sr, len(sizes), 2000, aptr, acols, exact_values(sr, rng, acols.size))
    st = {}
    got = esc_multiply(a, b, ctx=bins_ctx, stats=st)
    want = ob.orc_multiply(to_mat(a), to_mat(b))
    assert_same(got, want, sr)
    bins = st["rows_per_bin"]
    assert bins[0] == 2 and bins[1] >= 1 and bins[6] >= 1, bins
    assert sum(bins[2:6]) + bins[8] + bins[9] >= 3


@pytest.mark.parametrize("sr", [1, 2, 4])
def test_rmat14_against_reference_checksum(golden, ctx, sr):
    m = generators.generate_rmat(sr, 12 if sr != 4 else 14, 16.0, 1)
    a = coo_to_csr(m)
    d = DeviceCsr.upload(ctx, a)
    st = {}
    c = local_multiply(d, d, stats=st)
    if sr == 4:
        assert c.nnz == int(golden["rmat14_4_c_nnz"][0])
        assert c.checksum() == int(golden["rmat14_4_c_csum"][0])
        assert np.array_equal(np.diff(c.download().rowptr), golden["rmat14_4_c_rownnz"])
    else:
        s, z, f, _ = ob.orc_stream(to_mat(a), to_mat(a))
        assert c.nnz == z and st["products"] == f
        assert c.checksum() == (ob.orc_seed(a.nrows, a.ncols) + s) % (1 << 64)


@pytest.mark.parametrize("sr", [0, 2, 4, 5])
def test_output_modes_agree(bins_ctx, sr):
    """The three output strategies (U-slot scratch, exact claims, two passes)
    produce the same C; the scratch budget selects the strategy."""
    m = coo_to_csr(generators.generate_rmat(sr, 13, 16.0, 5))
    d = DeviceCsr.upload(bins_ctx, m)
    st = {}
    full = local_multiply(d, d, stats=st)
    assert st["output_mode"] == 0
    per = 4 + int(lib.spg_value_size(sr))
    want = full.download()
    for budget, mode in ((int(st["nnz_out"] * per * 1.02), 1), (1 << 20, 2)):
        bins_ctx.set_scratch_budget(budget)
        try:
            st2 = {}
            got = local_multiply(d, d, stats=st2)
        finally:
            bins_ctx.set_scratch_budget(0)
        assert st2["output_mode"] == mode
        assert_same(got.download(), want, sr, rtol=RTOL)


@pytest.mark.parametrize("sr", [0, 1, 2, 4, 5])
def test_merge_partials_matches_reference(golden, ctx, sr):
    parts = [unpack(golden, f"merge_{sr}_p{i}", sr) for i in range(4)]
    order = golden[f"merge_{sr}_order"]
    dparts = [DeviceCsr.upload(ctx, p) for p in parts]
    out = merge_partials(dparts, 40, 30, stages=order[0].tolist(), rounds=order[1].tolist())
    got = out.download()
    want = unpack(golden, f"merge_{sr}_c", sr, csc=True)
    assert isinstance(got, CscMatrix) and got.nrows == 40 and got.ncols == 30
    assert_same(got, want, sr)


def test_merge_extent_mismatch_is_internal_error(ctx):
    p = DeviceCsr.upload(ctx, CsrMatrix(4, 3, 4, np.zeros(4, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int32)))
    with pytest.raises(errors.InternalError):
        merge_partials([p], 5, 5)


def test_device_checksum_matches_reference(ctx):
    rng = np.random.default_rng(9)
    for sr in (0, 1, 2, 3, 4, 5):
        m = _rand(sr, rng, 77, 51, 0.1)
        assert matrix_checksum(m, ctx=ctx) == ob.orc_checksum(to_mat(m))


@pytest.mark.parametrize("sr", [0, 2, 4, 5])
def test_wide_output_uses_hash_bins(bins_ctx, sr):
    """Outputs wider than 16 dense panels with medium rows go to the hash bins."""
    rng = np.random.default_rng(7 + sr)
    from golden.make_golden import exact_values
    n = 1_200_000
    lens = rng.integers(30, 120, 400)
    bptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    bcols = np.concatenate([np.sort(rng.choice(n, L, replace=False)) for L in lens]).astype(np.int64)
    b = CsrMatrix(sr, 400, n, bptr, bcols, exact_values(sr, rng, bcols.size))
    rows = [np.sort(rng.choice(400, s, replace=False)) for s in (10, 20, 40, 3, 0, 50, 150)]
    aptr = np.concatenate([[0], np.cumsum([len(x) for x in rows])]).astype(np.int64)
    acols = np.concatenate(rows).astype(np.int64)
    a = CsrMatrix(sr, len(rows), 400, aptr, acols, exact_values(sr, rng, acols.size))
    st = {}
    got = esc_multiply(a, b, ctx=bins_ctx, stats=st)
    assert_same(got, ob.orc_multiply(to_mat(a), to_mat(b)), sr)
    assert sum(st["rows_per_bin"][i] for i in (3, 4, 7)) >= 2, st["rows_per_bin"]


@pytest.mark.parametrize("sorted_rows", [False, True])
@pytest.mark.parametrize("sr", [1, 2, 4])
def test_merge_dense_panels_against_oracle(bins_ctx, sr, sorted_rows):
    """Merging long partial rows over a wide block takes the dense panel path
    with per-partial binary-searched panel bounds (or, PIPE_SORTED, the sort
    fallback of bin 11, folding in partial order); checked against the oracle
    product [I I I] . vstack(partials)."""
    if sorted_rows:
        bins_ctx.set_pipeline(bins_ctx.PIPE_SORTED)
    rng = np.random.default_rng(3)
    from golden.make_golden import exact_values
    nrows, ncols, K = 6, 200_000, 3
    parts = []
    for _ in range(K):
        rs = [np.sort(rng.choice(ncols, int(rng.integers(6000, 9000)), replace=False)) for _ in range(nrows)]
        ptr = np.concatenate([[0], np.cumsum([len(x) for x in rs])]).astype(np.int64)
        idx = np.concatenate(rs).astype(np.int64)
        parts.append(CsrMatrix(sr, nrows, ncols, ptr, idx, exact_values(sr, rng, idx.size)))
    dparts = [DeviceCsr.upload(bins_ctx, p) for p in parts]
    st = {}
    out = merge_partials(dparts, ncols, nrows, stats=st).download()  # CSC of C == CSR of C^T
    one = {0: 1.0, 1: 0.0, 2: 1, 4: 0}[sr]
    L = ob.Mat(sr, nrows, K * nrows, np.arange(0, K * nrows + 1, K),
               np.array([q * nrows + i for i in range(nrows) for q in range(K)]), np.full(K * nrows, one))
    R = ob.Mat(sr, K * nrows, ncols, np.concatenate([[0], np.cumsum(np.concatenate([np.diff(p.rowptr) for p in parts]))]),
               np.concatenate([p.colids for p in parts]), np.concatenate([p.values for p in parts]))
    want = ob.orc_multiply(L, R)
    assert np.array_equal(out.colptr, want.ptr) and np.array_equal(out.rowids, want.idx)
    assert out.values.tobytes() == want.vals.tobytes()
    assert st["rows_per_bin"][11 if sorted_rows else 6] == nrows


@pytest.mark.parametrize("N", [7, 24])
def test_config4_stencil27_fp64_against_oracle(ctx, N):
    """BASELINE config 4 family (3D 27-point Laplacian, fp64): totals equal the
    closed forms and C equals the oracle within the fp64
    tolerance (integer-valued, so in fact exactly)."""
    a = coo_to_csr(generators.generate_stencil27(0, N))
    st = {}
    got = esc_multiply(a, a, ctx=ctx, stats=st)
    assert st["products"] == (9 * N - 10) ** 3 and got.nnz == (5 * N - 6) ** 3
    want = ob.orc_multiply(to_mat(a), to_mat(a))
    assert_same(got, want, 0, rtol=RTOL)
    assert np.array_equal(np.asarray(ptr_idx_vals(got)[2]), np.asarray(ptr_idx_vals(want)[2]))  # integer-valued: exact


@pytest.mark.parametrize("n,d", [(4096, 16), (1 << 14, 64)])
def test_config5_er_maxtimes_struct_against_oracle(ctx, n, d):
    """BASELINE config 5 family (ER rows, max-times on the {weight, tag}
    struct, value_mode 1): bit-exact against the oracle."""
    a = coo_to_csr(generators.generate_er(5, n, d, 1, value_mode=1))
    got = esc_multiply(a, a, ctx=ctx)
    want = ob.orc_multiply(to_mat(a), to_mat(a))
    assert_same(got, want, 5)


@pytest.mark.parametrize("sr", [1, 2, 4])
def test_bitrank_and_rank_panel_bins_against_oracle(bins_ctx, sr):
    """Rows sized for the bit-rank bin (2048 < F <= 8192) and the rank-panel
    bin (8192 < F <= 16384) over a 200K-column output: bit-exact vs the
    oracle (the other rows take the hash / dense bins)."""
    rng = np.random.default_rng(7 + sr)
    ncols, nb = 200_000, 64
    lens = np.full(nb, 1000)
    bptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    bcols = np.concatenate([np.sort(rng.choice(ncols, 1000, replace=False)) for _ in range(nb)]).astype(np.int64)
    from golden.make_golden import exact_values
    b = CsrMatrix(sr, nb, ncols, bptr, bcols, exact_values(sr, rng, bcols.size))
    rows = [np.sort(rng.choice(nb, k, replace=False)) for k in (3, 6, 12, 15, 16)]
    aptr = np.concatenate([[0], np.cumsum([len(x) for x in rows])]).astype(np.int64)
    acols = np.concatenate(rows).astype(np.int64)
    a = CsrMatrix(sr, len(rows), nb, aptr, acols, exact_values(sr, rng, acols.size))
    st = {}
    got = esc_multiply(a, b, ctx=bins_ctx, stats=st)
    assert_same(got, ob.orc_multiply(to_mat(a), to_mat(b)), sr)
    bins = st["rows_per_bin"]
    # 4-byte values: bit-rank (F <= 8192) + rank panels (F <= 16384); others: bit-rank only
    assert bins[8] + bins[9] >= (3 if int(lib.spg_value_size(sr)) == 4 else 1), bins


def test_bitrank_drops_columns_whose_products_are_all_zero(bins_ctx):
    """Tropical (min, saturating +): products that saturate to INT32_MAX are
    the semiring zero and must vanish from C (local_spgemm.hpp:57-58) — the
    bit-rank bin marks presence from columns alone and must redo such rows."""
    rng = np.random.default_rng(11)
    ncols, nb = 100_000, 8
    bptr = np.arange(0, 1000 * nb + 1, 1000, dtype=np.int64)
    bcols = np.concatenate([np.sort(rng.choice(ncols, 1000, replace=False)) for _ in range(nb)]).astype(np.int64)
    big = (1 << 30) + 5
    bvals = rng.integers(1, 100, bcols.size).astype(np.int32)
    bvals[: 2000] = big                      # B rows 0-1: saturate against a big A entry
    b = CsrMatrix(4, nb, ncols, bptr, bcols, bvals)
    acols = np.arange(nb, dtype=np.int64)
    avals = np.full(nb, 3, dtype=np.int32)
    avals[:2] = big                          # row 0 x B rows 0-1: all products saturate
    a = CsrMatrix(4, 1, nb, np.array([0, nb], dtype=np.int64), acols, avals)
    st = {}
    got = esc_multiply(a, b, ctx=bins_ctx, stats=st)
    want = ob.orc_multiply(to_mat(a), to_mat(b))
    assert_same(got, want, 4)
    assert st["rows_per_bin"][8] == 1


@pytest.mark.parametrize("sr", [2, 4])
def test_row_batched_multiply_concatenates_to_the_full_product(ctx, sr):
    """spg_local_multiply_rows: row windows of A (x) B (the row-batched form
    used to stream C out of HBM) concatenate to the full product."""
    import ctypes as C
    from paper_2504_06408_b200._lib import DCsr, MultStats, check
    a = coo_to_csr(generators.generate_rmat(sr, 12, 16.0, 2))
    d = DeviceCsr.upload(ctx, a)
    full = local_multiply(d, d).download()
    cuts = [0, 1, 700, 701, 2500, a.nrows]
    ptr, idx, vals = [np.zeros(1, np.int64)], [], []
    for r0, r1 in zip(cuts[:-1], cuts[1:]):
        out = DCsr()
        check(lib.spg_local_multiply_rows(ctx.handle, sr, C.byref(d.d), C.byref(d.d), r0, r1, C.byref(out),
                                          C.byref(MultStats())), ctx.handle)
        part = DeviceCsr(ctx, sr, out).download()
        assert part.nrows == r1 - r0
        ptr.append(part.rowptr[1:] + ptr[-1][-1])
        idx.append(part.colids)
        vals.append(part.values)
    assert np.array_equal(np.concatenate(ptr), full.rowptr)
    assert np.array_equal(np.concatenate(idx), full.colids)
    assert np.concatenate(vals).tobytes() == full.values.tobytes()


@pytest.mark.parametrize("sr,ncols", [(4, 40000), (4, 12000), (0, 20000)])
def test_heavy_and_dense_rows_share_the_chunk_table(bins_ctx, sr, ncols):
    """Per-bin pipeline, U-slot mode: heavy dense rows (F > 262144, the
    1-CTA/SM kernel with W-wide panels and 32 warps) and ordinary dense rows
    (2-CTA kernel, W/2 panels, 16 warps) write per-warp chunk tables of
    different sizes into one table — widths that are not a multiple of the
    panel width used to overflow it."""
    rng = np.random.default_rng(21)
    from golden.make_golden import exact_values
    nb = 64
    lens = np.full(nb, min(ncols // 2, 9000))
    bptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    bcols = np.concatenate([np.sort(rng.choice(ncols, L, replace=False)) for L in lens]).astype(np.int64)
    b = CsrMatrix(sr, nb, ncols, bptr, bcols, exact_values(sr, rng, bcols.size))
    rows = [np.arange(nb), np.arange(0, nb, 2), np.arange(5), np.arange(40)]  # F = 64 * L (heavy), ..., 5 * L
    aptr = np.concatenate([[0], np.cumsum([len(x) for x in rows])]).astype(np.int64)
    acols = np.concatenate(rows).astype(np.int64)
    a = CsrMatrix(sr, len(rows), nb, aptr, acols, exact_values(sr, rng, acols.size))
    st = {}
    got = esc_multiply(a, b, ctx=bins_ctx, stats=st)
    assert_same(got, ob.orc_multiply(to_mat(a), to_mat(b)), sr, rtol=RTOL if sr == 0 else None)
    assert st["rows_per_bin"][6] >= 2 and st["output_mode"] == 0, st


BIN_WIDE = 11


@pytest.mark.parametrize("sr", [0, 3, 5])
def test_wide_rows_sort_fallback_at_4m_columns(ctx, sr):
    """Rows with more distinct outputs than the largest shared-memory hash
    (> 4096 for 8/16-byte values) over 4 M columns, where the dense panels'
    per-segment offsets no longer fit shared memory (ER max-times at 1x1):
    the products are sorted in HBM and folded in the reference's order
    (bin 11), next to ordinary hash rows.  Overlapping right-operand rows make
    duplicates; fp64 uses non-integer values."""
    rng = np.random.default_rng(31 + sr)
    from golden.make_golden import exact_values
    ncols, nb, blen = 1 << 22, 80, 100
    pool = np.sort(rng.choice(ncols, 12000, replace=False))
    b_cols = [np.sort(rng.choice(pool, blen, replace=False)) for _ in range(nb)]
    bptr = np.concatenate([[0], np.cumsum([len(x) for x in b_cols])]).astype(np.int64)
    bc = np.concatenate(b_cols).astype(np.int64)
    bv = rng.standard_normal(bc.size) if sr == 0 else exact_values(sr, rng, bc.size)
    b = CsrMatrix(sr, nb, ncols, bptr, bc, bv)
    rows = [np.arange(nb), np.arange(0, nb, 2), np.arange(10), np.zeros(0, np.int64), np.arange(70)]
    aptr = np.concatenate([[0], np.cumsum([len(x) for x in rows])]).astype(np.int64)
    ac = np.concatenate(rows).astype(np.int64)
    av = rng.standard_normal(ac.size) if sr == 0 else exact_values(sr, rng, ac.size)
    a = CsrMatrix(sr, len(rows), nb, aptr, ac, av)
    st = {}
    got = esc_multiply(a, b, ctx=ctx, stats=st)
    assert_same(got, ob.orc_multiply(to_mat(a), to_mat(b)), sr, rtol=RTOL if sr == 0 else None)
    assert st["rows_per_bin"][BIN_WIDE] >= 2, st["rows_per_bin"]


@pytest.mark.parametrize("sr", [0, 1, 2, 4, 5])
def test_sorted_pipeline_equals_oracle_on_dense_rows(ctx, sr):
    """PIPE_SORTED sends every dense-panel row through the sort fallback:
    long R-MAT rows (with exact cancellations possible for fp64) must give
    the same C as the oracle, in every output mode the fallback serves."""
    m = coo_to_csr(generators.generate_rmat(sr, 12, 16.0, 4))
    d = DeviceCsr.upload(ctx, m)
    ctx.set_pipeline(ctx.PIPE_SORTED)
    try:
        st = {}
        got = local_multiply(d, d, stats=st).download()
        assert st["rows_per_bin"][BIN_WIDE] > 0 and st["rows_per_bin"][6] == 0, st["rows_per_bin"]
        ctx.set_scratch_budget(1 << 20)  # exact-claim / two-pass modes
        st2 = {}
        got2 = local_multiply(d, d, stats=st2).download()
        assert st2["output_mode"] in (1, 2)
    finally:
        ctx.set_pipeline(ctx.PIPE_AUTO)
        ctx.set_scratch_budget(0)
    want = ob.orc_multiply(to_mat(m), to_mat(m))
    assert_same(got, want, sr, rtol=RTOL if sr == 0 else None)
    assert_same(got2, want, sr, rtol=RTOL if sr == 0 else None)


def test_download_with_split_index_widening():
    """The host result's int64 column indices come back in 2^25-entry chunks,
    a share widened on the GPU (crossing PCIe as int64) and the rest widened
    by host threads from int32 staging (SPG_D2H_GPU_WIDEN=0.5 here, read once
    per process): the host C equals the device C (checksum of the uploaded
    host result vs the device checksum)."""
    import os
    import subprocess
    import sys
    code = """
import sys
from paper_2504_06408_b200 import Context, DeviceCsr, esc_multiply, generators, local_multiply, matrix_checksum
a = generators.coo_to_csr_fast(generators.generate_rmat(4, 16, 16.0, 3))
ctx = Context(0)
c = esc_multiply(a, a, ctx=ctx)
assert c.nnz > 2 * (1 << 25), c.nnz
d = DeviceCsr.upload(ctx, a)
dc = local_multiply(d, d)
assert matrix_checksum(c, ctx) == dc.checksum()
print("ok", c.nnz)
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {**os.environ, "SPG_D2H_GPU_WIDEN": "0.5", "PYTHONPATH": root}
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr


@pytest.mark.parametrize("sr", [0, 4, 5])
def test_optimistic_small_hash_and_overflow_rerun(bins_ctx, sr):
    """2K-slot bin rows (512 < F <= 1024) run first in a 512-slot table: rows
    with <= 256 distinct columns finish there, rows with more stop inserting
    and are re-run in the 2K table — both kinds side by side, against the
    oracle."""
    rng = np.random.default_rng(77 + sr)
    from golden.make_golden import exact_values
    ncols, nb, blen = 1_000_000, 40, 25  # column spans > 2^18: no bit-rank window
    narrow = np.sort(rng.choice(ncols, 200, replace=False))
    b_cols = [np.sort(rng.choice(narrow if k < nb // 2 else ncols, blen, replace=False)) for k in range(nb)]
    bptr = np.concatenate([[0], np.cumsum([len(x) for x in b_cols])]).astype(np.int64)
    bc = np.concatenate(b_cols).astype(np.int64)
    b = CsrMatrix(sr, nb, ncols, bptr, bc, exact_values(sr, rng, bc.size))
    lo, hi = np.arange(nb // 2), np.arange(nb // 2, nb)
    # F = 550 / 550 / 525 products; <= 250, ~500, <= 225 distinct columns
    rows = [np.concatenate([lo, hi[:2]]), np.concatenate([lo[:2], hi]), np.concatenate([lo, hi[:1]])]
    aptr = np.concatenate([[0], np.cumsum([len(x) for x in rows])]).astype(np.int64)
    ac = np.concatenate(rows).astype(np.int64)
    a = CsrMatrix(sr, len(rows), nb, aptr, ac, exact_values(sr, rng, ac.size))
    st = {}
    got = esc_multiply(a, b, ctx=bins_ctx, stats=st)
    assert_same(got, ob.orc_multiply(to_mat(a), to_mat(b)), sr, rtol=RTOL if sr == 0 else None)
    assert st["rows_per_bin"][5] == 3, st["rows_per_bin"]
    nnz = np.diff(got.rowptr)
    assert nnz[0] <= 256 < nnz[1]  # one row fits the small table, one overflows


def test_large_upload_narrows_on_host_and_checks_range(ctx):
    """Uploads of >= 2^22 indices cross PCIe as int32, narrowed and
    range-checked by host threads (two chunks of 2^25 here): the device matrix
    equals the host one, and an index outside the block raises
    MalformedInputError as the device narrowing does."""
    rng = np.random.default_rng(8)
    n, ncols, per = 1 << 20, 1 << 22, 40
    ptr = np.arange(0, n * per + 1, per, dtype=np.int64)
    idx = np.sort(rng.integers(0, ncols, (n, per)), axis=1).reshape(-1).astype(np.int64)
    vals = rng.integers(0, 100, idx.size).astype(np.int32)
    m = CsrMatrix(4, n, ncols, ptr, idx, vals)
    got = DeviceCsr.upload(ctx, m).download()
    assert np.array_equal(got.colids, idx) and np.array_equal(got.rowptr, ptr)
    bad = idx.copy()
    bad[idx.size - 7] = ncols  # one column id past the block
    with pytest.raises(errors.MalformedInputError):
        DeviceCsr.upload(ctx, CsrMatrix(4, n, ncols, ptr, bad, vals))
