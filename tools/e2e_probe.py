import sys, time
sys.path.insert(0, '.')
from paper_2504_06408_b200 import generators, esc_multiply
from paper_2504_06408_b200.device import pin
a = generators.coo_to_csr_fast(generators.permute_symmetric(generators.generate_rmat(4, 18, 16.0, 1), 1))
pin(a.rowptr, a.colids, a.values)
for r in range(3):
    t0 = time.perf_counter(); c = esc_multiply(a, a); print("e2e", r, time.perf_counter() - t0, file=sys.stderr); del c
