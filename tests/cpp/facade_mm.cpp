// CPU-only use of the facade's read_matrix_market<SR> (matrix_market.hpp:43-141):
// prints "nrows ncols nnz" then one "row col value" line per tuple, or
// "error <class> <message>" when the reader throws.
#include <cstdio>

#include "spsumma_b200.hpp"

using namespace spsumma_b200;

int main(int argc, char** argv) {
  if (argc < 2) return 2;
  try {
    const auto m = read_matrix_market<ArithmeticSemiring>(argv[1]);
    std::printf("%lld %lld %lld\n", (long long)m.nrows, (long long)m.ncols, (long long)m.tuples.size());
    for (const auto& t : m.tuples) std::printf("%lld %lld %.17g\n", (long long)t.row, (long long)t.col, t.value);
  } catch (const UnsupportedFormatError& e) {
    std::printf("error UnsupportedFormatError %s\n", e.what());
  } catch (const MalformedInputError& e) {
    std::printf("error MalformedInputError %s\n", e.what());
  }
  return 0;
}
