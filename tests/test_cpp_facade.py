"""The reference-shaped C++ facade (include/spsumma_b200.hpp): it compiles and
links against libspgemm_b200.so on CPU; on the GPU its results match the
oracle bit-exactly."""
import os
import subprocess

import numpy as np
import pytest

import oracle_bind as ob

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "build", "facade_main")


def build_facade(src="facade_main.cpp", exe=BIN):
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    lib_dir = os.path.join(ROOT, "paper_2504_06408_b200")
    cmd = ["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", src), "-o", exe, "-L", lib_dir, "-lspgemm_b200",
           f"-Wl,-rpath,{lib_dir}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_facade_compiles_and_links():
    assert os.path.exists(build_facade())


@pytest.mark.gpu
def test_facade_matches_oracle():
    exe = build_facade()
    out = subprocess.run([exe, "10"], check=True, capture_output=True, text=True).stdout
    kv = dict(x.split("=") for x in out.split())
    from paper_2504_06408_b200 import generators
    from paper_2504_06408_b200.formats import coo_to_csr
    a = coo_to_csr(generators.generate_rmat(4, 10, 16.0, 1))
    want = ob.orc_multiply(ob.Mat.of(a), ob.Mat.of(a))
    assert int(kv["nnz"]) == want.nnz
    assert int(kv["checksum"]) == ob.orc_checksum(want)
    assert int(kv["merge_nnz"]) == want.nnz
    assert kv["shape_error"] == "1"


def test_facade_read_matrix_market(tmp_path):
    """read_matrix_market<SR> through the C++ facade (no GPU): tuples and the
    exception classes of matrix_market.hpp."""
    exe = build_facade("facade_mm.cpp", os.path.join(ROOT, "build", "facade_mm"))
    good = tmp_path / "g.mtx"
    good.write_text("%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n1 1 2.5\n3 1 -1\n3 1 4\n")
    out = subprocess.run([exe, str(good)], check=True, capture_output=True, text=True).stdout.split("\n")
    assert out[:4] == ["3 3 3", "0 0 2.5", "0 2 3", "2 0 3"]
    bad = tmp_path / "b.mtx"
    bad.write_text("%%MatrixMarket matrix array real general\n1 1\n1\n")
    out = subprocess.run([exe, str(bad)], check=True, capture_output=True, text=True).stdout
    assert out.startswith("error UnsupportedFormatError ") and "unsupported format 'array'" in out
    bad.write_text("%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1\n")
    out = subprocess.run([exe, str(bad)], check=True, capture_output=True, text=True).stdout
    assert out.strip() == f"error MalformedInputError {bad}:3: file ends after 1 of 2 entries"


def test_summa_facade_compiles_and_links():
    assert os.path.exists(build_facade("summa_facade_main.cpp", os.path.join(ROOT, "build", "summa_facade_main")))


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 4])
def test_summa_facade_matches_reference(golden, p):
    """summa25_multiply(DistMatrix, DistMatrix, LatencyModel, CommConfig,
    SummaOptions) -> SummaResult through the facade, one thread per rank:
    gather(product) and the ledger's per-instance counters equal the
    reference's summa25_multiply on the same input (golden section 6)."""
    exe = build_facade("summa_facade_main.cpp", os.path.join(ROOT, "build", "summa_facade_main"))
    out = subprocess.run([exe, str(p), "9", "8", "3", "0"], check=True, capture_output=True, text=True,
                         timeout=600).stdout
    kv = dict(x.split("=") for x in out.split())
    key = f"summa_4_p{p}_r1"
    led = golden[key + "_ledger"]
    assert int(kv["checksum"]) == int(golden[key + "_csum"][0])
    assert int(kv["nnz"]) == int(golden[key + "_nnz"][0])
    assert int(kv["bcasts"]) == int(led[0] + led[1])
    assert int(kv["size_exchanges"]) == int(led[4])
    assert int(kv["multiplies"]) == int(led[5])
    assert int(kv["skipped"]) == int(led[6])
    assert kv["grid_error"] == "1"
