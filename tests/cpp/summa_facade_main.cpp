// The reference's distributed API through the facade (include/spsumma_b200.hpp),
// written the way a reference user writes it (tools/spsumma.cpp:201-204):
//   distribute(A, ProcessGrid(p)) -> summa25_multiply(A, A, model, cfg, opts)
//   -> gather(result.product) -> matrix_checksum
// Prints "p=<p> nnz=<n> checksum=<c> bcasts=<b> size_exchanges=<s>
// multiplies=<m> skipped=<k> grid_error=<0|1>" for tests/test_cpp_facade.py.
#include <cstdio>

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
  for (const auto& t : m.tuples) {
    out.colids.push_back(t.col);
    out.values.push_back(t.value);
  }
  return out;
}

int main(int argc, char** argv) {
  const int p = argc > 1 ? std::atoi(argv[1]) : 4;
  const int scale = argc > 2 ? std::atoi(argv[2]) : 9;
  const double ef = argc > 3 ? std::atof(argv[3]) : 8.0;
  const int seed = argc > 4 ? std::atoi(argv[4]) : 3;
  const int fuse = argc > 5 ? std::atoi(argv[5]) : 0;
  const auto coo = generate_rmat<SR>(scale, ef, seed);
  const auto a = distribute(coo, ProcessGrid(p));
  CommConfig cfg;
  cfg.mode = CommMode::host_only;  // ranks may share one GPU in the test
  SummaOptions opts;
  opts.fuse_stages = fuse != 0;
  const auto res = summa25_multiply(a, a, LatencyModel::bundled_default(), cfg, opts);
  const auto c = gather(res.product);
  const auto cs = matrix_checksum(default_context(), to_csr(c));
  bool grid_error = false;
  try {
    ProcessGrid bad(3);
  } catch (const GridError&) {
    grid_error = true;
  }
  std::printf("p=%d nnz=%lld checksum=%llu bcasts=%llu size_exchanges=%llu multiplies=%llu skipped=%llu grid_error=%d\n",
              p, (long long)c.tuples.size(), (unsigned long long)cs,
              (unsigned long long)(res.ledger.host_bcasts + res.ledger.device_bcasts),
              (unsigned long long)res.ledger.size_exchanges, (unsigned long long)res.ledger.local_multiply_calls,
              (unsigned long long)res.ledger.skipped_stages, grid_error ? 1 : 0);
  return 0;
}
