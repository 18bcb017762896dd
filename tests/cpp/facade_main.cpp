// Exercises the reference-shaped C++ facade (include/spsumma_b200.hpp) the way
// a reference user would: generate_rmat -> CSR -> esc_multiply -> checksum,
// merge_partials of two partials, and the error mapping.  Prints one line
// "nnz=<n> checksum=<c> merge_nnz=<m>" for tests/test_cpp_facade.py.
#include <cstdio>
#include <map>

#include "spsumma_b200.hpp"

using namespace spsumma_b200;
using SR = TropicalI32Semiring;

static CsrMatrix<SR> to_csr(const CooMatrix<SR>& m) {
  CsrMatrix<SR> out;
  out.nrows = m.nrows;
  out.ncols = m.ncols;
  out.rowptr.assign((size_t)m.nrows + 1, 0);
  for (const auto& t : m.tuples) ++out.rowptr[(size_t)t.row + 1];
  for (index_t r = 0; r < m.nrows; ++r) out.rowptr[(size_t)r + 1] += out.rowptr[(size_t)r];
  for (const auto& t : m.tuples) {  // tuples are normalised: row-major, unique
    out.colids.push_back(t.col);
    out.values.push_back(t.value);
  }
  return out;
}

int main(int argc, char** argv) {
  const int scale = argc > 1 ? std::atoi(argv[1]) : 10;
  Context ctx(0);
  const auto a = to_csr(generate_rmat<SR>(scale, 16.0, 1));
  const auto c = esc_multiply(ctx, a, a);
  const auto cs = matrix_checksum(ctx, c);
  // merge two copies of C^T-shaped partials: min(x, x) = x, so the merge is C itself (as CSC)
  std::vector<Partial<SR>> parts{{0, 0, c}, {0, 1, c}};
  const auto merged = merge_partials(ctx, parts, c.ncols, c.nrows);
  bool threw = false;
  try {
    CsrMatrix<SR> bad;
    bad.nrows = 3;
    bad.ncols = 3;
    bad.rowptr.assign(4, 0);
    esc_multiply(ctx, a, bad);
  } catch (const ShapeError&) {
    threw = true;
  }
  std::printf("nnz=%lld checksum=%llu merge_nnz=%lld shape_error=%d\n", (long long)c.nnz(),
              (unsigned long long)cs, (long long)merged.nnz(), threw ? 1 : 0);
  return 0;
}
