"""CPU: Matrix Market ingestion against the
reference's read_matrix_market (matrix_market.hpp:43-141, run through
oracle/_ref): same normalised COO for every semiring, same error class and
message on malformed and unsupported files.  One GPU case multiplies a read
matrix and checks it against the oracle."""
import numpy as np
import pytest

import oracle_bind as ob
from paper_2504_06408_b200 import errors, read_matrix_market
from paper_2504_06408_b200.matrix_market import verify_corpus
from paper_2504_06408_b200.semiring import SemiringId

GOOD = {
    "general_real": "%%MatrixMarket matrix coordinate real general\n% comment\n4 5 6\n1 1 1.5\n2 3 -2.25\n"
                    "4 5 1e3\n2 3 2.25\n1 1 0.5\n3 2 0\n",
    "symmetric_int": "%%MatrixMarket matrix coordinate integer symmetric\n\n%c\n   \n3 3 4\n1 1 7\n3 1 2\n"
                     "2 1 -5\n3 3 1\n",
    "pattern_sym": "%%MATRIXMARKET Matrix Coordinate Pattern Symmetric\n5 5 5\n1 2\n2 1\n5 5\n4 2\n  3   1  \n",
    "pattern_general_crlf": "%%MatrixMarket matrix coordinate pattern general\r\n3 4 3\r\n3 4\r\n1 1\r\n3 4\r\n",
    "prefix_numbers": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 2 3.5abc\n2x 1 +4\n",
    "empty": "%%MatrixMarket matrix coordinate real general\n0 0 0\n",
    "trailing_ignored": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 9\n2 2 8\n",
    "tiny_values": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1e-300\n1 1 -1e-300\n2 1 0.001\n",
}
BAD = {
    "empty_file": "",
    "no_header": "3 3 1\n1 1 1\n",
    "short_header": "%%MatrixMarket matrix coordinate real\n1 1 1\n1 1 1\n",
    "array": "%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "vector": "%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n",
    "bad_size": "%%MatrixMarket matrix coordinate real general\n3 3\n1 1 1\n",
    "no_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n\n",
    "nonnumeric_size": "%%MatrixMarket matrix coordinate real general\na 3 1\n1 1 1\n",
    "negative_size": "%%MatrixMarket matrix coordinate real general\n-1 3 1\n1 1 1\n",
    "field_count": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1\n",
    "pattern_field_count": "%%MatrixMarket matrix coordinate pattern general\n3 3 1\n1 1 1\n",
    "nonnumeric_entry": "%%MatrixMarket matrix coordinate real general\n3 3 1\n1 1 x\n",
    "out_of_range": "%%MatrixMarket matrix coordinate real general\n3 3 1\n4 1 1\n",
    "zero_index": "%%MatrixMarket matrix coordinate real general\n3 3 1\n0 1 1\n",
    "truncated": "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 1 1\n2 2 2\n",
    "overflow": "%%MatrixMarket matrix coordinate real general\n3 3 1\n99999999999999999999 1 1\n",
}
STATUS_CLASS = {5: errors.MalformedInputError, 14: errors.UnsupportedFormatError}

needs_ref = pytest.mark.skipif(ob.ref is None, reason="oracle/_ref not built (needs /root/reference)")


def _write(tmp_path, name, text):
    p = tmp_path / f"{name}.mtx"
    p.write_bytes(text.encode())
    return str(p)


@needs_ref
@pytest.mark.parametrize("name", sorted(GOOD))
@pytest.mark.parametrize("sr", [SemiringId.arithmetic, SemiringId.minplus, SemiringId.boolean,
                                SemiringId.minselect, SemiringId.tropical_i32, SemiringId.maxtimes])
def test_reader_matches_reference(tmp_path, name, sr):
    path = _write(tmp_path, name, GOOD[name])
    rc, msg, want = ob.ref_read_matrix_market(int(sr), path)
    assert rc == 0, msg
    got = read_matrix_market(sr, path)
    nr, nc, r, c, v = want
    assert (got.nrows, got.ncols) == (nr, nc)
    assert np.array_equal(got.rows, r) and np.array_equal(got.cols, c)
    assert got.values.tobytes() == v.tobytes()


@needs_ref
@pytest.mark.parametrize("name", sorted(BAD))
def test_errors_match_reference(tmp_path, name):
    path = _write(tmp_path, name, BAD[name])
    rc, msg, _ = ob.ref_read_matrix_market(int(SemiringId.arithmetic), path)
    assert rc in STATUS_CLASS, (rc, msg)
    with pytest.raises(STATUS_CLASS[rc]) as ei:
        read_matrix_market("arithmetic", path)
    assert str(ei.value) == msg


def test_reader_known_answer(tmp_path):
    # symmetric integer file: mirrored off-diagonals, duplicates folded, sorted
    m = read_matrix_market("arithmetic", _write(tmp_path, "s", GOOD["symmetric_int"]))
    assert (m.nrows, m.ncols) == (3, 3)
    assert m.rows.tolist() == [0, 0, 0, 1, 2, 2]
    assert m.cols.tolist() == [0, 1, 2, 0, 0, 2]
    assert m.values.tolist() == [7.0, -5.0, 2.0, -5.0, 2.0, 1.0]
    # general real: (2,3) folds -2.25 + 2.25 = 0 and is dropped; stored 0 dropped
    g = read_matrix_market("arithmetic", _write(tmp_path, "g", GOOD["general_real"]))
    assert list(zip(g.rows.tolist(), g.cols.tolist(), g.values.tolist())) == [(0, 0, 2.0), (3, 4, 1000.0)]
    with pytest.raises(errors.MalformedInputError, match=r"missing\.mtx: cannot open file"):
        read_matrix_market("arithmetic", str(tmp_path / "missing.mtx"))


def test_verify_corpus_lines(tmp_path):
    lines = []
    p = _write(tmp_path, "atmosmodd_small", GOOD["general_real"])
    q = _write(tmp_path, "other", GOOD["general_real"])
    assert verify_corpus([p, q], out=lines.append) == 1
    assert lines[0].startswith(f"FAIL {p}: expected 1270432x1270432 nnz 8814880, found 4x5 nnz 2")
    assert lines[1] == f"SKIP {q} (not a known corpus matrix)"
    assert lines[2].startswith("PASS rmat generator (65536x65536, nnz ")
    assert lines[3:] == ["SKIP delaunay (no file supplied)", "SKIP long (no file supplied)"]


@pytest.mark.gpu
def test_read_then_multiply_on_gpu(tmp_path, ctx):
    from paper_2504_06408_b200 import DeviceCsr, local_multiply
    from paper_2504_06408_b200.formats import coo_to_csr
    rng = np.random.default_rng(5)
    n, k = 300, 2400
    r, c = rng.integers(1, n + 1, k), rng.integers(1, n + 1, k)
    v = rng.integers(-9, 10, k)
    body = "".join(f"{a} {b} {x}\n" for a, b, x in zip(r, c, v))
    path = _write(tmp_path, "rand", f"%%MatrixMarket matrix coordinate integer symmetric\n{n} {n} {k}\n{body}")
    for sr in (SemiringId.arithmetic, SemiringId.tropical_i32):
        a = coo_to_csr(read_matrix_market(sr, path))
        d = DeviceCsr.upload(ctx, a)
        got = local_multiply(d, d).download()
        want = ob.orc_multiply(ob.Mat.of(a), ob.Mat.of(a))
        assert np.array_equal(got.rowptr, want.ptr) and np.array_equal(got.colids, want.idx)
        if sr == SemiringId.arithmetic:
            np.testing.assert_allclose(got.values, want.vals, rtol=1e-12)
        else:
            assert got.values.tobytes() == want.vals.tobytes()
