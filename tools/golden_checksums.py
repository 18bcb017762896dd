"""Golden matrix_checksum values of C = A.A for the BASELINE configs that
bench.py checks its own C against, computed with the CPU oracle's streaming
restatement (oracle/spg_oracle.cpp, pinned to the reference by
tests/test_oracle.py) on all host cores.  Test infrastructure: run here, not
on the GPU box; the printed values are committed into bench.GOLDEN_CSUM.

  python tools/golden_checksums.py 4 252     # config 4: stencil N
  python tools/golden_checksums.py 5 22 64 1 # config 5: ER 2^log2, d, seed
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle_bind as ob  # noqa: E402
from paper_2504_06408_b200 import generators  # noqa: E402


def main():
    cfg = int(sys.argv[1])
    t0 = time.time()
    if cfg == 4:
        N = int(sys.argv[2])
        coo = generators.generate_stencil27(0, N)
        key = (4, N)
    elif cfg == 5:
        log2, d, seed = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
        coo = generators.generate_er(5, 1 << log2, d, seed, value_mode=1)
        key = (5, log2, d, seed)
    else:
        raise SystemExit("config 4 or 5")
    a = generators.coo_to_csr_fast(coo)
    del coo
    m = ob.Mat.of(a)
    t1 = time.time()
    s, z, f, _ = ob.orc_stream(m, m, nthreads=os.cpu_count() or 8)
    csum = (ob.orc_seed(a.nrows, a.ncols) + s) % (1 << 64)
    print(f"{key}: {csum},  # nnz(C) = {z}, products = {f}; "
          f"generate {t1 - t0:.0f} s, oracle {time.time() - t1:.0f} s", flush=True)


if __name__ == "__main__":
    main()
