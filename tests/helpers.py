"""Shared test helpers: golden-fixture unpacking and exact/tolerance compares."""
import numpy as np

import oracle_bind as ob
from paper_2504_06408_b200.formats import CsrMatrix, CscMatrix

# fp64 (+, x) tolerance: pattern exact, |x-y| <= 1e-12 max(|x|,|y|) + 1e-300
RTOL = 1e-12


def unpack(g, prefix, sr, csc=False):
    nr, nc = (int(x) for x in g[prefix + "_dims"])
    cls = CscMatrix if csc else CsrMatrix
    return cls(sr, nr, nc, g[prefix + "_ptr"].astype(np.int64), g[prefix + "_idx"].astype(np.int64),
               g[prefix + "_vals"])


def ptr_idx_vals(m):
    if hasattr(m, "rowptr"):
        return m.rowptr, m.colids, m.values
    if hasattr(m, "colptr"):
        return m.colptr, m.rowids, m.values
    return m.ptr, m.idx, m.vals


def assert_same(got, want, sr, rtol=None):
    """Pattern bit-exact; values bit-exact unless sr is arithmetic (tolerance)."""
    gp, gi, gv = ptr_idx_vals(got)
    wp, wi, wv = ptr_idx_vals(want)
    assert np.array_equal(np.asarray(gp), np.asarray(wp)), "row/col pointers differ"
    assert np.array_equal(np.asarray(gi), np.asarray(wi)), "indices differ"
    gv, wv = np.asarray(gv), np.asarray(wv)
    if int(sr) == 0 and rtol is not None:
        diff = np.abs(gv - wv)
        bound = rtol * np.maximum(np.abs(gv), np.abs(wv)) + 1e-300
        assert np.all(diff <= bound), f"max rel err {np.max(diff / np.maximum(np.abs(wv), 1e-300))}"
    else:
        assert gv.tobytes() == wv.tobytes(), "values differ"


def to_mat(m):
    return ob.Mat.of(m)
