"""Regenerates the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists and oracle/_ref/
libspsumma_ref.so was compiled from its unmodified headers):

    python tests/golden/make_golden.py

Every expected output below is produced by the reference's own functions
(esc_multiply, naive_multiply, generate_rmat, random_coo, merge_partials,
summa25_multiply + gather, matrix_checksum, find_crossover), so the fixtures
pin parity to the reference, not to the oracle restatement.  The GPU box has
no /root/reference: tests there read these committed files.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_bind as ob  # noqa: E402

SEMIRINGS = [0, 1, 2, 3, 4, 5]


def exact_values(sr, rng, n):
    """Integer-valued draws (testutil ValueGen exact=true analogue), so any
    fold grouping gives bit-identical results."""
    if sr == 0:
        return rng.integers(1, 17, n).astype(np.float64)
    if sr == 1:
        return rng.integers(1, 11, n).astype(np.float64)
    if sr == 2:
        return np.ones(n, dtype=np.uint8)
    if sr == 3:
        v = np.zeros(n, dtype=ob._DT[3])
        v["weight"] = rng.integers(1, 11, n)
        v["payload"] = rng.integers(0, 100, n)
        return v
    if sr == 4:
        return rng.integers(1, 2048, n).astype(np.int32)
    v = np.zeros(n, dtype=ob._DT[5])
    v["w"] = rng.integers(1, 8, n).astype(np.float64)
    v["tag"] = rng.integers(0, 1 << 62, n, dtype=np.uint64)
    return v


def random_csr(sr, rng, nrows, ncols, density):
    mask = rng.random((nrows, ncols)) < density
    r, c = np.nonzero(mask)
    vals = exact_values(sr, rng, r.size)
    return ob.ref_coo_to_csr(sr, nrows, ncols, r, c, vals)


def pack(prefix, m: ob.Mat, d: dict):
    d[prefix + "_dims"] = np.array([m.nrows, m.ncols], dtype=np.int64)
    d[prefix + "_ptr"] = m.ptr
    d[prefix + "_idx"] = m.idx
    d[prefix + "_vals"] = m.vals


def main():
    assert ob.ref is not None, "oracle/_ref/libspsumma_ref.so is required (make -C oracle)"
    rng = np.random.default_rng(20250406)
    d = {}

    # 1. local multiply: every semiring, square and rectangular, several densities
    cases = []
    for sr in SEMIRINGS:
        for (m, k, n, dens) in [(64, 64, 64, 0.08), (37, 53, 29, 0.15), (96, 96, 96, 0.02), (16, 16, 16, 0.5)]:
            a = random_csr(sr, rng, m, k, dens)
            b = random_csr(sr, rng, k, n, dens)
            c = ob.ref_esc(a, b)
            c_naive = ob.ref_naive(a, b)
            assert np.array_equal(c.ptr, c_naive.ptr) and np.array_equal(c.idx, c_naive.idx)
            key = f"mul_{sr}_{m}x{k}x{n}"
            pack(key + "_a", a, d)
            pack(key + "_b", b, d)
            pack(key + "_c", c, d)
            d[key + "_csum"] = np.array([ob.ref_checksum(c)], dtype=np.uint64)
            cases.append(key)
    d["mul_cases"] = np.array(cases)

    # 2. SPEC examples
    a = ob.Mat(0, 2, 2, [0, 2, 3], [0, 1, 1], np.array([1.0, 2.0, 3.0]))
    pack("spec_aa", ob.ref_esc(a, a), d)
    w = ob.Mat(1, 3, 3, [0, 2, 4, 5], [0, 1, 1, 2, 2], np.array([0.0, 1.0, 0.0, 2.0, 0.0]))
    pack("spec_ww", ob.ref_esc(w, w), d)

    # 3. generators: R-MAT s10 ef16 per semiring, reference tuples
    for sr in (0, 1, 2, 4):
        nr, nc, r, c, v = ob.ref_generate_rmat(sr, 10, 16.0, 1)
        d[f"rmat10_{sr}_rows"] = r
        d[f"rmat10_{sr}_cols"] = c
        d[f"rmat10_{sr}_vals"] = v
    # R-MAT s14 (tropical) summary: nnz + checksum of A and of esc(A, A)
    nr, nc, r, c, v = ob.ref_generate_rmat(4, 14, 16.0, 1)
    A = ob.ref_coo_to_csr(4, nr, nc, r, c, v)
    d["rmat14_4_a_nnz"] = np.array([A.nnz], dtype=np.int64)
    d["rmat14_4_a_csum"] = np.array([ob.ref_checksum(A)], dtype=np.uint64)
    C14 = ob.ref_esc(A, A)
    d["rmat14_4_c_nnz"] = np.array([C14.nnz], dtype=np.int64)
    d["rmat14_4_c_csum"] = np.array([ob.ref_checksum(C14)], dtype=np.uint64)
    d["rmat14_4_c_rownnz"] = np.diff(C14.ptr)

    # 4. config 1: testutil random_coo<Arithmetic>(42, 4096, 4096, 8/4096, exact=false)
    nr, nc, r, c, v = ob.ref_random_coo(0, 42, 4096, 4096, 8.0 / 4096, exact=False)
    d["er4096_rows"], d["er4096_cols"], d["er4096_vals"] = r, c, v
    A = ob.ref_coo_to_csr(0, nr, nc, r, c, v)
    C1 = ob.ref_esc(A, A)
    pack("er4096_c", C1, d)

    # 5. merge_partials (summa.hpp:122-172): 4 partials of a 40 x 30 C block
    for sr in SEMIRINGS:
        if sr == 3:
            continue
        parts = [random_csr(sr, rng, 30, 40, 0.1) for _ in range(4)]
        stages, rounds = [1, 0, 1, 0], [0, 1, 1, 0]
        out = ob.ref_merge(parts, stages, rounds, 40, 30)
        for i, p in enumerate(parts):
            pack(f"merge_{sr}_p{i}", p, d)
        d[f"merge_{sr}_order"] = np.array([stages, rounds], dtype=np.int32)
        pack(f"merge_{sr}_c", out, d)

    # 6. distributed reference results: gather(summa25_multiply) checksums and ledgers
    for sr in (1, 2, 4):
        nr, nc, r, c, v = ob.ref_generate_rmat(sr, 9, 8.0, 3)
        for p in (1, 4, 9):
            for two in (1, 0):
                rc, coo, cs, led = ob.ref_summa(sr, nr, nc, r, c, v, p, two_round=two, mode=2, threshold=4096)
                assert rc == 0
                d[f"summa_{sr}_p{p}_r{two}_csum"] = np.array([cs], dtype=np.uint64)
                d[f"summa_{sr}_p{p}_r{two}_ledger"] = np.array(led)
                d[f"summa_{sr}_p{p}_r{two}_nnz"] = np.array([coo[2].size], dtype=np.int64)

    # 7. find_crossover on the bundled model (tuner.hpp:17-39)
    d["crossover"] = np.array([ob.ref_find_crossover(f, 1, 1 << 30) for f in (2, 3, 4, 8)], dtype=np.int64)

    # 8. row/col slices (summa.hpp:57-98)
    m = random_csr(4, rng, 50, 70, 0.1)
    pack("slice_m", m, d)
    pack("slice_rows", ob.ref_slice(m, True, 7, 31), d)
    pack("slice_cols", ob.ref_slice(m, False, 13, 52), d)

    out = os.path.join(HERE, "golden.npz")
    np.savez_compressed(out, **d)
    print(f"wrote {out}: {os.path.getsize(out) / 1e6:.2f} MB, {len(d)} arrays")


if __name__ == "__main__":
    main()
