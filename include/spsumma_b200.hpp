// spsumma_b200.hpp — reference-shaped C++ facade over the C-ABI.
//
// A user of the reference library (/root/reference/proj/include/spsumma)
// switches by including this header instead of the reference headers and
// linking libspgemm_b200.so; names, argument meaning and the exception
// classes follow the reference:
//
//   reference                                   this facade
//   -----------------------------------------   ----------------------------------
//   SemiringLike + built-ins (semiring.hpp)      tag types with the same names
//   CooMatrix/CscMatrix/DcscMatrix/CsrMatrix     same structs (std::vector-backed)
//     (formats.hpp:16-86)
//   esc_multiply(a, b, chunk) (local_spgemm:83)  esc_multiply(a, b)  -> GPU
//   merge_partials (summa.hpp:122-172)           merge_partials(...)  -> GPU
//   matrix_checksum (checksum.hpp:20-38)         matrix_checksum(...) -> GPU
//   generate_rmat (rmat.hpp:15-60)               generate_rmat<SR>(...) (bit-identical)
//   summa25_multiply (summa.hpp:248-349)         summa25_multiply(comm, ...) — one
//                                                rank per process/GPU (torchrun/MPI
//                                                style), returns this rank's C block
//   Error / ShapeError / ... (common.hpp:12-73)  same class names, thrown from the
//                                                C-ABI status codes
//
// Only the built-in semirings have device instantiations in the shipped
// library; a custom semiring is added by SPG_INSTANTIATE in a user .cu file
// (paper_2504_06408_b200/csrc/instantiate.cuh).
#pragma once
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "spgemm_b200.h"

namespace spsumma_b200 {

using index_t = std::int64_t;

// ------------------------------------------------------------ exceptions
class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class MalformedInputError : public Error { public: using Error::Error; };
class UnsupportedFormatError : public Error { public: using Error::Error; };
class ShapeError : public Error { public: using Error::Error; };
class GridError : public Error { public: using Error::Error; };
class UnsupportedSemiringError : public Error { public: using Error::Error; };
class ProtocolError : public Error { public: using Error::Error; };
class DeadlockError : public Error { public: using Error::Error; };
class AbortedError : public Error { public: using Error::Error; };
class InvalidRangeError : public Error { public: using Error::Error; };
class InternalError : public Error { public: using Error::Error; };
class DeviceError : public Error { public: using Error::Error; };

inline void throw_status(int st, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (st) {
    case SPG_OK: return;
    case SPG_ERR_SHAPE: throw ShapeError(m);
    case SPG_ERR_GRID: throw GridError(m);
    case SPG_ERR_UNSUPPORTED_SEMIRING: throw UnsupportedSemiringError(m);
    case SPG_ERR_PROTOCOL: case SPG_ERR_NCCL: throw ProtocolError(m);
    case SPG_ERR_MALFORMED: throw MalformedInputError(m);
    case SPG_ERR_UNSUPPORTED_FORMAT: throw UnsupportedFormatError(m);
    case SPG_ERR_INVALID_RANGE: throw InvalidRangeError(m);
    case SPG_ERR_INTERNAL: throw InternalError(m);
    case SPG_ERR_ABORTED: throw AbortedError(m);
    case SPG_ERR_DEADLOCK: throw DeadlockError(m);
    default: throw DeviceError(m);
  }
}

// Throws for a failed C-ABI status, reading the message only AFTER the call
// returned (the message pointer is invalidated by the call that sets it, so
// it must not be an argument evaluated alongside that call).
inline void throw_last(int st) {
  if (st != SPG_OK) throw_status(st, spg_last_error(nullptr));
}

// -------------------------------------------------------------- semirings
struct MinSelect {
  double weight = __builtin_huge_val();
  std::int64_t payload = INT64_MAX;
  bool operator==(const MinSelect&) const = default;
};
struct MaxTimesValue {
  double w = 0.0;
  std::uint64_t tag = 0;
  bool operator==(const MaxTimesValue&) const = default;
};
// Tag types: value_type + C-ABI id (semiring.hpp:43-120 semantics on device).
struct ArithmeticSemiring { using value_type = double; static constexpr int id = SPG_SR_ARITHMETIC; static constexpr bool is_commutative_mul = true; };
struct MinPlusSemiring { using value_type = double; static constexpr int id = SPG_SR_MINPLUS; static constexpr bool is_commutative_mul = true; };
struct BooleanSemiring { using value_type = std::uint8_t; static constexpr int id = SPG_SR_BOOLEAN; static constexpr bool is_commutative_mul = true; };
struct MinSelectSemiring { using value_type = MinSelect; static constexpr int id = SPG_SR_MINSELECT; static constexpr bool is_commutative_mul = false; };
struct TropicalI32Semiring { using value_type = std::int32_t; static constexpr int id = SPG_SR_TROPICAL_I32; static constexpr bool is_commutative_mul = true; };
struct MaxTimesSemiring { using value_type = MaxTimesValue; static constexpr int id = SPG_SR_MAXTIMES; static constexpr bool is_commutative_mul = true; };

// ---------------------------------------------------------------- formats
template <class SR>
struct CooMatrix {
  using value_type = typename SR::value_type;
  struct Tuple { index_t row = 0, col = 0; value_type value{}; };
  index_t nrows = 0, ncols = 0;
  std::vector<Tuple> tuples;
  index_t nnz() const { return (index_t)tuples.size(); }
};
template <class SR>
struct CscMatrix {
  using value_type = typename SR::value_type;
  index_t nrows = 0, ncols = 0;
  std::vector<index_t> colptr{0}, rowids;
  std::vector<value_type> values;
  index_t nnz() const { return (index_t)rowids.size(); }
};
template <class SR>
struct DcscMatrix {
  using value_type = typename SR::value_type;
  index_t nrows = 0, ncols = 0;
  std::vector<index_t> jc, cp{0}, rowids;
  std::vector<value_type> values;
  index_t nnz() const { return (index_t)rowids.size(); }
};
template <class SR>
struct CsrMatrix {
  using value_type = typename SR::value_type;
  index_t nrows = 0, ncols = 0;
  std::vector<index_t> rowptr{0}, colids;
  std::vector<value_type> values;
  index_t nnz() const { return (index_t)colids.size(); }
};

namespace detail {
template <class M>
spg_hcsr view_csr(const M& m) {
  spg_hcsr h{m.nrows, m.ncols, m.nnz(), const_cast<index_t*>(m.rowptr.data()),
             const_cast<index_t*>(m.colids.data()), const_cast<void*>(static_cast<const void*>(m.values.data()))};
  return h;
}
template <class M>
spg_hcsr view_csc(const M& m) {
  spg_hcsr h{m.nrows, m.ncols, m.nnz(), const_cast<index_t*>(m.colptr.data()),
             const_cast<index_t*>(m.rowids.data()), const_cast<void*>(static_cast<const void*>(m.values.data()))};
  return h;
}
template <class V>
void take(std::vector<V>& dst, void* src, index_t n) {
  dst.resize((size_t)n);
  if (n) std::memcpy(dst.data(), src, sizeof(V) * (size_t)n);
}
inline void take_idx(std::vector<index_t>& dst, index_t* src, index_t n) {
  dst.assign(src, src + n);
}
}  // namespace detail

// ------------------------------------------------------------------ context
class Context {
 public:
  explicit Context(int device = 0) { throw_last(spg_ctx_create(device, &c_)); }
  ~Context() { spg_ctx_destroy(c_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  spg_ctx* get() const { return c_; }
  void check(int st) const { throw_status(st, spg_last_error(c_)); }

 private:
  spg_ctx* c_ = nullptr;
};

// --------------------------------------------------------- local operators
// esc_multiply(a, b) (local_spgemm.hpp:83-156): GPU multiply of host CSR operands.
template <class SR>
CsrMatrix<SR> esc_multiply(Context& ctx, const CsrMatrix<SR>& a, const CsrMatrix<SR>& b,
                           spg_mult_stats* stats = nullptr) {
  spg_hcsr ha = detail::view_csr(a), hb = detail::view_csr(b), hc{};
  ctx.check(spg_esc_multiply(ctx.get(), SR::id, &ha, &hb, &hc, stats));
  CsrMatrix<SR> out;
  out.nrows = hc.nrows;
  out.ncols = hc.ncols;
  detail::take_idx(out.rowptr, hc.ptr, hc.nrows + 1);
  detail::take_idx(out.colids, hc.idx, hc.nnz);
  detail::take(out.values, hc.vals, hc.nnz);
  spg_hcsr_free(&hc);
  return out;
}

// matrix_checksum (checksum.hpp:20-38) of a CSR, computed on the GPU.
template <class SR>
std::uint64_t matrix_checksum(Context& ctx, const CsrMatrix<SR>& m) {
  spg_hcsr h = detail::view_csr(m);
  spg_dcsr d{};
  ctx.check(spg_upload(ctx.get(), SR::id, &h, 0, &d));
  std::uint64_t out = 0;
  const int st = spg_checksum(ctx.get(), SR::id, &d, 0, &out);
  spg_dcsr_free(ctx.get(), &d);
  ctx.check(st);
  return out;
}

// Partial for merge_partials (summa.hpp:109-116): a C^T partial as host CSR.
template <class SR>
struct Partial {
  int stage = 0;
  int round = 0;
  CsrMatrix<SR> ct;
};

// merge_partials (summa.hpp:122-172): GPU merge into the CSC C block.
template <class SR>
CscMatrix<SR> merge_partials(Context& ctx, const std::vector<Partial<SR>>& parts, index_t block_rows,
                             index_t block_cols) {
  std::vector<spg_dcsr> dp(parts.size());
  std::vector<int> stages, rounds;
  int st = SPG_OK;
  size_t up = 0;
  for (; up < parts.size() && st == SPG_OK; ++up) {
    spg_hcsr h = detail::view_csr(parts[up].ct);
    st = spg_upload(ctx.get(), SR::id, &h, 0, &dp[up]);
    stages.push_back(parts[up].stage);
    rounds.push_back(parts[up].round);
  }
  spg_dcsr out{};
  if (st == SPG_OK)
    st = spg_merge_partials(ctx.get(), SR::id, (int)parts.size(), dp.data(), stages.data(), rounds.data(),
                            block_rows, block_cols, &out, nullptr);
  for (size_t k = 0; k < up; ++k) spg_dcsr_free(ctx.get(), &dp[k]);
  ctx.check(st);
  spg_hcsr h{};
  st = spg_download(ctx.get(), SR::id, &out, 1, &h);
  spg_dcsr_free(ctx.get(), &out);
  ctx.check(st);
  CscMatrix<SR> c;
  c.nrows = h.nrows;
  c.ncols = h.ncols;
  detail::take_idx(c.colptr, h.ptr, h.ncols + 1);
  detail::take_idx(c.rowids, h.idx, h.nnz);
  detail::take(c.values, h.vals, h.nnz);
  spg_hcsr_free(&h);
  return c;
}

// generate_rmat<SR>(scale, edge_factor, seed) (rmat.hpp:15-60), bit-identical.
template <class SR>
CooMatrix<SR> generate_rmat(int scale, double edge_factor, std::uint64_t seed) {
  int64_t n = 0, nnz = 0;
  int64_t *rows = nullptr, *cols = nullptr;
  void* vals = nullptr;
  throw_last(spg_generate_rmat(SR::id, scale, edge_factor, seed, &n, &nnz, &rows, &cols, &vals));
  CooMatrix<SR> out;
  out.nrows = out.ncols = n;
  out.tuples.resize((size_t)nnz);
  const auto* v = static_cast<const typename SR::value_type*>(vals);
  for (int64_t k = 0; k < nnz; ++k) out.tuples[k] = {rows[k], cols[k], v[k]};
  spg_free(rows);
  spg_free(cols);
  spg_free(vals);
  return out;
}

// read_matrix_market<SR>(path) (matrix_market.hpp:43-141): normalised COO.
template <class SR>
CooMatrix<SR> read_matrix_market(const std::string& path) {
  int64_t m = 0, n = 0, nnz = 0;
  int64_t *rows = nullptr, *cols = nullptr;
  void* vals = nullptr;
  throw_last(spg_read_matrix_market(SR::id, path.c_str(), &m, &n, &nnz, &rows, &cols, &vals));
  CooMatrix<SR> out;
  out.nrows = m;
  out.ncols = n;
  out.tuples.resize((size_t)nnz);
  const auto* v = static_cast<const typename SR::value_type*>(vals);
  for (int64_t k = 0; k < nnz; ++k) out.tuples[k] = {rows[k], cols[k], v[k]};
  spg_free(rows);
  spg_free(cols);
  spg_free(vals);
  return out;
}

// ---------------------------------------------------------- distributed
// One rank of a pr x pc grid (rank = i * pc + j), one process per GPU.
class Comm {
 public:
  Comm(const std::string& job, int world, int rank, int pr, int pc, int device,
       std::uint64_t staging_bytes = 64ull << 20) {
    const int st = spg_comm_create(job.c_str(), world, rank, pr, pc, device, staging_bytes, &c_);
    if (st != SPG_OK) throw_status(st, spg_comm_last_error(nullptr));
  }
  ~Comm() { spg_comm_destroy(c_); }
  Comm(const Comm&) = delete;
  Comm& operator=(const Comm&) = delete;
  spg_comm* get() const { return c_; }

 private:
  spg_comm* c_ = nullptr;
};

enum class CommMode { host_only = SPG_COMM_HOST_ONLY, device_only = SPG_COMM_DEVICE_ONLY, hybrid = SPG_COMM_HYBRID };
struct CommConfig {  // comm.hpp:36-39
  CommMode mode = CommMode::hybrid;
  std::uint64_t threshold_bytes = 0;
};
struct SummaOptions {  // summa.hpp:174-177 (chunk_nnz has no GPU meaning)
  bool two_round = true;
  bool fuse_stages = true;  // one fused multiply over all received panels (no merge)
};

// summa25_multiply for this rank's blocks (CSC or DCSC, LocalBlock layout).
// Returns this rank's C block (CSC, host) and fills the ledger.
template <class SR>
CscMatrix<SR> summa25_multiply(Comm& comm, Context& ctx, index_t a_nrows, index_t a_ncols, index_t b_ncols,
                               const CscMatrix<SR>& a_block, const CscMatrix<SR>& b_block,
                               const CommConfig& cfg = {}, const SummaOptions& opts = {},
                               spg_ledger* ledger = nullptr) {
  spg_hcsr ha = detail::view_csc(a_block), hb = detail::view_csc(b_block);
  spg_summa_opts o{opts.two_round ? 1 : 0, static_cast<int>(cfg.mode), cfg.threshold_bytes, 0,
                   opts.fuse_stages ? 1 : 0};
  spg_dcsr c{};
  ctx.check(spg_summa25_multiply(comm.get(), ctx.get(), SR::id, a_nrows, a_ncols, b_ncols, &ha, nullptr, &hb,
                                 nullptr, &o, &c, ledger));
  spg_hcsr h{};
  const int st = spg_download(ctx.get(), SR::id, &c, 1, &h);
  spg_dcsr_free(ctx.get(), &c);
  ctx.check(st);
  CscMatrix<SR> out;
  out.nrows = h.nrows;
  out.ncols = h.ncols;
  detail::take_idx(out.colptr, h.ptr, h.ncols + 1);
  detail::take_idx(out.rowids, h.idx, h.nnz);
  detail::take(out.values, h.vals, h.nnz);
  spg_hcsr_free(&h);
  return out;
}

}  // namespace spsumma_b200
