import sys; sys.path.insert(0,'tests')
import numpy as np, oracle_bind as ob
from helpers import to_mat
from paper_2504_06408_b200.formats import CsrMatrix
from golden.make_golden import exact_values
sr=0
rng = np.random.default_rng(31 + sr)
ncols, nb, blen = 1 << 22, 80, 100
pool = np.sort(rng.choice(ncols, 12000, replace=False))
b_cols = [np.sort(rng.choice(pool, blen, replace=False)) for _ in range(nb)]
bptr = np.concatenate([[0], np.cumsum([len(x) for x in b_cols])]).astype(np.int64)
bc = np.concatenate(b_cols).astype(np.int64)
bv = rng.standard_normal(bc.size)
b = CsrMatrix(sr, nb, ncols, bptr, bc, bv)
rows = [np.arange(nb), np.arange(0, nb, 2), np.arange(10), np.zeros(0, np.int64), np.arange(70)]
aptr = np.concatenate([[0], np.cumsum([len(x) for x in rows])]).astype(np.int64)
ac = np.concatenate(rows).astype(np.int64)
av = rng.standard_normal(ac.size)
a = CsrMatrix(sr, len(rows), nb, aptr, ac, av)

from paper_2504_06408_b200 import esc_multiply, Context
import faulthandler; faulthandler.enable()
ctx = Context(0)
print("gpu...", flush=True)
st = {}
got = esc_multiply(a, b, ctx=ctx, stats=st)
print("done", got.nnz, st["rows_per_bin"], flush=True)
