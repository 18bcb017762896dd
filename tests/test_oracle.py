"""CPU: the parity oracle (oracle/spg_oracle.cpp) is pinned to the reference.

Every expected value here comes from the reference's own functions, either
through the committed golden fixtures (tests/golden/make_golden.py) or live
through oracle/_ref (the reference compiled from its unmodified headers).
"""
import numpy as np
import pytest

import oracle_bind as ob
from helpers import RTOL, assert_same

pytestmark = pytest.mark.skipif(ob.orc is None, reason="oracle/liboracle.so not built (make -C oracle)")


def mat(g, key, sr):
    nr, nc = (int(x) for x in g[key + "_dims"])
    return ob.Mat(sr, nr, nc, g[key + "_ptr"], g[key + "_idx"], g[key + "_vals"])


def test_oracle_matches_reference_esc_on_all_golden_cases(golden):
    for key in golden["mul_cases"]:
        sr = int(str(key).split("_")[1])
        a, b, want = mat(golden, key + "_a", sr), mat(golden, key + "_b", sr), mat(golden, key + "_c", sr)
        got = ob.orc_multiply(a, b)
        # exact integer-valued draws: bit-exact for every semiring
        assert_same(got, want, sr)
        assert ob.orc_checksum(got) == int(golden[key + "_csum"][0])


def test_oracle_spec_examples(golden):
    # SPEC.md:244  A = [[1,2],[0,3]]  =>  A.A = [[1,8],[0,9]]
    a = ob.Mat(0, 2, 2, [0, 2, 3], [0, 1, 1], np.array([1.0, 2.0, 3.0]))
    got = ob.orc_multiply(a, a)
    assert got.ptr.tolist() == [0, 2, 3] and got.idx.tolist() == [0, 1, 1]
    assert got.vals.tolist() == [1.0, 8.0, 9.0]
    assert_same(got, mat(golden, "spec_aa", 0), 0)
    # SPEC.md:246  min-plus 2-hop (W.W)[0][2] = 3
    w = ob.Mat(1, 3, 3, [0, 2, 4, 5], [0, 1, 1, 2, 2], np.array([0.0, 1.0, 0.0, 2.0, 0.0]))
    ww = ob.orc_multiply(w, w)
    row0 = dict(zip(ww.idx[ww.ptr[0]:ww.ptr[1]].tolist(), ww.vals[ww.ptr[0]:ww.ptr[1]].tolist()))
    assert row0[2] == 3.0
    assert_same(ww, mat(golden, "spec_ww", 1), 1)


def test_oracle_config1_er4096_fp64(golden):
    r, c, v = golden["er4096_rows"], golden["er4096_cols"], golden["er4096_vals"]
    assert r.size == 32763
    order = np.lexsort((c, r))
    ptr = np.concatenate([[0], np.cumsum(np.bincount(r, minlength=4096))])
    a = ob.Mat(0, 4096, 4096, ptr, c[order], v[order])
    got = ob.orc_multiply(a, a)
    want = mat(golden, "er4096_c", 0)
    assert want.nnz == 259911
    # the oracle folds in ascending k like esc_multiply: bit-exact here too
    assert_same(got, want, 0, rtol=RTOL)


def test_oracle_stream_checksum_equals_full():
    for sr in (0, 1, 2, 4, 5):
        rng = np.random.default_rng(sr)
        n = 300
        mask = rng.random((n, n)) < 0.05
        rr, cc = np.nonzero(mask)
        from golden.make_golden import exact_values
        vals = exact_values(sr, rng, rr.size)
        ptr = np.concatenate([[0], np.cumsum(np.bincount(rr, minlength=n))])
        a = ob.Mat(sr, n, n, ptr, cc, vals)
        full = ob.orc_multiply(a, a)
        s, z, f, rn = ob.orc_stream(a, a, rownnz=True)
        assert z == full.nnz
        assert np.array_equal(rn, np.diff(full.ptr))
        assert (ob.orc_seed(n, n) + s) % (1 << 64) == ob.orc_checksum(full)


@pytest.mark.skipif(ob.ref is None, reason="reference harness not built")
def test_oracle_matches_reference_on_rmat14_tropical(golden):
    nr, nc, r, c, v = ob.ref_generate_rmat(4, 14, 16.0, 1)
    a = ob.ref_coo_to_csr(4, nr, nc, r, c, v)
    assert a.nnz == int(golden["rmat14_4_a_nnz"][0])
    s, z, f, rn = ob.orc_stream(a, a, rownnz=True)
    assert z == int(golden["rmat14_4_c_nnz"][0])
    assert (ob.orc_seed(nr, nc) + s) % (1 << 64) == int(golden["rmat14_4_c_csum"][0])
    assert np.array_equal(rn, golden["rmat14_4_c_rownnz"])


@pytest.mark.skipif(ob.ref is None, reason="reference harness not built")
def test_oracle_checksum_matches_reference_checksum():
    rng = np.random.default_rng(5)
    for sr in (0, 1, 2, 3, 4, 5):
        from golden.make_golden import random_csr
        m = random_csr(sr, rng, 40, 33, 0.2)
        assert ob.orc_checksum(m) == ob.ref_checksum(m)
        csc = ob.Mat(sr, m.ncols, m.nrows, m.ptr, m.idx, m.vals, csc=True)  # CSR read as CSC of the transpose
        assert ob.orc_checksum(csc) == ob.ref_checksum(csc)
