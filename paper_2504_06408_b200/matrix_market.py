"""read_matrix_market<SR>(path) (proj/include/spsumma/matrix_market.hpp:43-141).

The parser is host C++ inside the library (csrc/mm.cu, spg_read_matrix_market);
this is the reference-shaped call: ASCII coordinate files (real / integer /
pattern, general / symmetric) -> normalised COO (formats.hpp:105-133).
MalformedInputError "path:line: what" for structural errors,
UnsupportedFormatError for headers the reader does not handle.
"""
from __future__ import annotations

import ctypes as C
import os

from ._lib import check, lib
from .formats import CooMatrix
from .generators import _take
from .semiring import as_id


def read_matrix_market(sr, path) -> CooMatrix:
    sr = as_id(sr)
    nrows, ncols, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    rows, cols = C.POINTER(C.c_int64)(), C.POINTER(C.c_int64)()
    vals = C.c_void_p()
    check(lib.spg_read_matrix_market(int(sr), os.fsencode(path), C.byref(nrows), C.byref(ncols), C.byref(nnz),
                                     C.byref(rows), C.byref(cols), C.byref(vals)))
    r, c, v = _take(sr, nnz.value, rows, cols, vals)
    return CooMatrix(int(sr), nrows.value, ncols.value, r, c, v)


# Evaluation corpus shapes (tools/spsumma.cpp:253-263): key, rows, cols, nnz (0: dims only).
CORPUS = (
    ("atmosmodd", 1270432, 1270432, 8814880),
    ("delaunay_n22", 4194304, 4194304, 25165738),
    ("delaunay_n23", 8388608, 8388608, 0),
    ("long_dt_coup0", 1470152, 1470152, 70219816),
    ("long_coup_dt0", 1470152, 1470152, 70219816),
)


def verify_corpus(files, out=print) -> int:
    """cmd_verify_corpus (tools/spsumma.cpp:253-321): PASS/FAIL/SKIP lines per
    file against the corpus table, plus the R-MAT generator dimension check;
    returns 1 if any check failed, else 0."""
    from .generators import generate_rmat
    failed = False
    seen = []
    for path in files:
        stem = os.path.basename(path).lower()
        row = next((k for k in CORPUS if k[0] in stem), None)
        if row is None:
            out(f"SKIP {path} (not a known corpus matrix)")
            continue
        key, nr, nc, nz = row
        seen.append(key)
        m = read_matrix_market("arithmetic", path)
        if m.nrows == nr and m.ncols == nc and (nz == 0 or m.nnz == nz):
            out(f"PASS {path} ({m.nrows}x{m.ncols}, nnz {m.nnz})")
        else:
            failed = True
            exp = f"{nr}x{nc}" + (f" nnz {nz}" if nz else "")
            out(f"FAIL {path}: expected {exp}, found {m.nrows}x{m.ncols} nnz {m.nnz}")
    g = generate_rmat("arithmetic", 16, 7.5, 1)
    if g.nrows == 65536 and g.ncols == 65536:
        out(f"PASS rmat generator (65536x65536, nnz {g.nnz})")
    else:
        failed = True
        out(f"FAIL rmat generator: dimensions {g.nrows}x{g.ncols}, expected 65536x65536")
    for key in ("atmosmodd", "delaunay", "long"):
        if not any(key in s for s in seen):
            out(f"SKIP {key} (no file supplied)")
    return 1 if failed else 0
