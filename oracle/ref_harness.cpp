// TEST INFRASTRUCTURE — NOT PRODUCT CODE.
//
// C-ABI harness around the UNMODIFIED reference library.  It #includes the
// header-only reference from /root/reference/proj/include (never copied into
// this repo) and is built by oracle/Makefile into oracle/_ref/libspsumma_ref.so.
// It serves two purposes:
//   1. pin the CPU restatement (oracle/spg_oracle.cpp) and the product's host
//      code (generators, slicing, schedule) to the reference's own behaviour
//      on golden inputs (tests/test_oracle.py, tests/test_host.py);
//   2. time the reference CPU path for bench.py's cpu_baseline leg and
//      `bench.py --impl reference`.
// The two semirings the reference lacks (TropicalI32 for BASELINE config 2,
// MaxTimes for config 5) are defined here as SemiringLike types with their
// ValueCodec specialisations, exactly as a reference user would add them
// (semiring.hpp:28-40, serialize.hpp:29-76).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "spsumma/checksum.hpp"
#include "spsumma/dist_matrix.hpp"
#include "spsumma/formats.hpp"
#include "spsumma/local_spgemm.hpp"
#include "spsumma/matrix_market.hpp"
#include "spsumma/rmat.hpp"
#include "spsumma/semiring.hpp"
#include "spsumma/serialize.hpp"
#include "spsumma/summa.hpp"
#include "spsumma/tuner.hpp"
#include "tests/testutil.hpp"  // the reference's own seeded fixture generators

namespace harness {

struct TropicalI32Semiring {
  using value_type = std::int32_t;
  static constexpr std::string_view name = "tropical_i32";
  static constexpr bool is_commutative_mul = true;
  static value_type add(value_type a, value_type b) { return std::min(a, b); }
  static value_type mul(value_type a, value_type b) {
    if (a == zero() || b == zero()) return zero();
    const std::int64_t s = std::int64_t{a} + std::int64_t{b};
    if (s >= std::int64_t{zero()}) return zero();
    if (s < std::numeric_limits<std::int32_t>::min()) return std::numeric_limits<std::int32_t>::min();
    return static_cast<value_type>(s);
  }
  static constexpr value_type zero() { return std::numeric_limits<std::int32_t>::max(); }
  static constexpr value_type one() { return 0; }
  static bool is_zero(value_type v) { return v == zero(); }
  // Fixed-point weights: 1/1024 resolution (SURVEY.md §8d config 2 note).
  static value_type from_real(double x) {
    const double y = x * 1024.0;
    if (!(y < 2147483646.5)) return zero();
    if (y < -2147483648.0) return std::numeric_limits<std::int32_t>::min();
    return static_cast<value_type>(std::llround(y));
  }
};

struct MaxTimesValue {
  double w = 0.0;
  std::uint64_t tag = 0;
  bool operator==(const MaxTimesValue&) const = default;
};

struct MaxTimesSemiring {
  using value_type = MaxTimesValue;
  static constexpr std::string_view name = "maxtimes";
  static constexpr bool is_commutative_mul = true;
  static value_type add(const value_type& a, const value_type& b) {
    return (b.w > a.w || (b.w == a.w && b.tag > a.tag)) ? b : a;
  }
  static value_type mul(const value_type& a, const value_type& b) {
    const double w = a.w * b.w;
    if (w == 0.0) return zero();
    return {w, a.tag ^ b.tag};
  }
  static value_type zero() { return {0.0, 0}; }
  static value_type one() { return {1.0, 0}; }
  static bool is_zero(const value_type& v) { return v.w == 0.0; }
  static value_type from_real(double x) { return {x, 0}; }
};

static_assert(spsumma::SemiringLike<TropicalI32Semiring>);
static_assert(spsumma::SemiringLike<MaxTimesSemiring>);

}  // namespace harness

namespace spsumma {
template <>
struct ValueCodec<std::int32_t> {
  static constexpr std::size_t size = 4;
  static void encode(std::int32_t v, std::byte* out) {
    const auto u = static_cast<std::uint32_t>(v);
    for (int i = 0; i < 4; ++i) out[i] = static_cast<std::byte>((u >> (8 * i)) & 0xff);
  }
  static std::int32_t decode(const std::byte* p) {
    std::uint32_t u = 0;
    for (int i = 0; i < 4; ++i) u |= std::uint32_t{std::to_integer<std::uint8_t>(p[i])} << (8 * i);
    return static_cast<std::int32_t>(u);
  }
};
template <>
struct ValueCodec<harness::MaxTimesValue> {
  static constexpr std::size_t size = 16;
  static void encode(const harness::MaxTimesValue& v, std::byte* out) {
    store_u64le(out, std::bit_cast<std::uint64_t>(v.w));
    store_u64le(out + 8, v.tag);
  }
  static harness::MaxTimesValue decode(const std::byte* p) {
    return {std::bit_cast<double>(load_u64le(p)), load_u64le(p + 8)};
  }
};
}  // namespace spsumma

using namespace spsumma;

extern "C" {
struct ref_csr {  // CSR (or CSC) with logical dims; ptr has nseg + 1 entries
  int64_t nrows, ncols, nnz;
  int64_t* ptr;
  int64_t* idx;
  void* vals;
};
struct ref_coo {
  int64_t nrows, ncols, nnz;
  int64_t* rows;
  int64_t* cols;
  void* vals;
};
}

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const GridError& e) {
    g_err = e.what();
    return 2;
  } catch (const UnsupportedSemiringError& e) {
    g_err = e.what();
    return 3;
  } catch (const ProtocolError& e) {
    g_err = e.what();
    return 4;
  } catch (const MalformedInputError& e) {
    g_err = e.what();
    return 5;
  } catch (const InvalidRangeError& e) {
    g_err = e.what();
    return 6;
  } catch (const InternalError& e) {
    g_err = e.what();
    return 7;
  } catch (const UnsupportedFormatError& e) {
    g_err = e.what();
    return 14;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

// Ids shared with the product and the oracle (include/spgemm_b200.h).
template <class F>
int with_ref_sr(int sr, F&& f) {
  switch (sr) {
    case 0: return f(std::type_identity<ArithmeticSemiring>{});
    case 1: return f(std::type_identity<MinPlusSemiring>{});
    case 2: return f(std::type_identity<BooleanSemiring>{});
    case 3: return f(std::type_identity<MinSelectSemiring>{});
    case 4: return f(std::type_identity<harness::TropicalI32Semiring>{});
    case 5: return f(std::type_identity<harness::MaxTimesSemiring>{});
  }
  g_err = "unknown semiring id";
  return 8;
}

template <class V>
constexpr std::size_t raw_size() {
  if constexpr (std::is_same_v<V, bool>) return 1;
  else return sizeof(V);
}

template <class V>
void load_vals(std::vector<V>& dst, const void* src, int64_t n) {
  dst.resize(static_cast<std::size_t>(n));
  if constexpr (std::is_same_v<V, bool>) {
    const auto* s = static_cast<const std::uint8_t*>(src);
    for (int64_t i = 0; i < n; ++i) dst[i] = s[i] != 0;
  } else {
    if (n) std::memcpy(dst.data(), src, sizeof(V) * n);
  }
}

template <class V>
void* store_vals(const std::vector<V>& src) {
  const std::size_t n = src.size();
  void* out = std::malloc(raw_size<V>() * std::max<std::size_t>(n, 1));
  if constexpr (std::is_same_v<V, bool>) {
    auto* d = static_cast<std::uint8_t*>(out);
    for (std::size_t i = 0; i < n; ++i) d[i] = src[i] ? 1 : 0;
  } else {
    if (n) std::memcpy(out, src.data(), sizeof(V) * n);
  }
  return out;
}

int64_t* store_idx(const std::vector<index_t>& v) {
  auto* out = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * std::max<std::size_t>(v.size(), 1)));
  if (!v.empty()) std::memcpy(out, v.data(), sizeof(int64_t) * v.size());
  return out;
}

template <class SR>
CsrMatrix<SR> to_csr(const ref_csr& m) {
  CsrMatrix<SR> out;
  out.nrows = m.nrows;
  out.ncols = m.ncols;
  out.rowptr.assign(m.ptr, m.ptr + m.nrows + 1);
  out.colids.assign(m.idx, m.idx + m.nnz);
  load_vals(out.values, m.vals, m.nnz);
  return out;
}

template <class SR>
CscMatrix<SR> to_csc(const ref_csr& m) {
  CscMatrix<SR> out;
  out.nrows = m.nrows;
  out.ncols = m.ncols;
  out.colptr.assign(m.ptr, m.ptr + m.ncols + 1);
  out.rowids.assign(m.idx, m.idx + m.nnz);
  load_vals(out.values, m.vals, m.nnz);
  return out;
}

template <class SR>
void from_csr(const CsrMatrix<SR>& m, ref_csr* out) {
  out->nrows = m.nrows;
  out->ncols = m.ncols;
  out->nnz = m.nnz();
  out->ptr = store_idx(m.rowptr);
  out->idx = store_idx(m.colids);
  out->vals = store_vals(m.values);
}

template <class SR>
void from_csc(const CscMatrix<SR>& m, ref_csr* out) {
  out->nrows = m.nrows;
  out->ncols = m.ncols;
  out->nnz = m.nnz();
  out->ptr = store_idx(m.colptr);
  out->idx = store_idx(m.rowids);
  out->vals = store_vals(m.values);
}

template <class SR>
CooMatrix<SR> to_coo(const ref_coo& m) {
  CooMatrix<SR> out;
  out.nrows = m.nrows;
  out.ncols = m.ncols;
  std::vector<typename SR::value_type> vals;
  load_vals(vals, m.vals, m.nnz);
  out.tuples.resize(static_cast<std::size_t>(m.nnz));
  for (int64_t i = 0; i < m.nnz; ++i) out.tuples[i] = {m.rows[i], m.cols[i], vals[i]};
  return out;
}

template <class SR>
void from_coo(const CooMatrix<SR>& m, ref_coo* out) {
  out->nrows = m.nrows;
  out->ncols = m.ncols;
  out->nnz = m.nnz();
  std::vector<index_t> r(m.tuples.size()), c(m.tuples.size());
  std::vector<typename SR::value_type> v(m.tuples.size());
  for (std::size_t i = 0; i < m.tuples.size(); ++i) {
    r[i] = m.tuples[i].row;
    c[i] = m.tuples[i].col;
    v[i] = m.tuples[i].value;
  }
  out->rows = store_idx(r);
  out->cols = store_idx(c);
  out->vals = store_vals(v);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

// generate_rmat<SR>(scale, edge_factor, seed), rmat.hpp:15-60.
int ref_generate_rmat(int sr, int scale, double edge_factor, uint64_t seed, ref_coo* out) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      from_coo(generate_rmat<SR>(scale, edge_factor, seed), out);
      return 0;
    });
  });
}

// read_matrix_market<SR>(path), matrix_market.hpp:43-141.
int ref_read_matrix_market(int sr, const char* path, ref_coo* out) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      from_coo(read_matrix_market<SR>(path), out);
      return 0;
    });
  });
}

// testutil::random_coo<SR>(mt19937_64(seed), n, m, density, exact)
// (proj/tests/testutil.hpp:58-73): the reference's own fixture generator;
// BASELINE config 1 is random_coo<Arithmetic>(42, 4096, 4096, 8/4096, false).
int ref_random_coo(int sr, uint64_t seed, int64_t nrows, int64_t ncols, double density, int exact,
                   ref_coo* out) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      if constexpr (std::is_same_v<SR, harness::TropicalI32Semiring> ||
                    std::is_same_v<SR, harness::MaxTimesSemiring>) {
        g_err = "random_coo has no ValueGen for this semiring";
        return 8;
      } else {
        std::mt19937_64 rng(seed);
        from_coo(testutil::random_coo<SR>(rng, nrows, ncols, density, exact != 0), out);
        return 0;
      }
    });
  });
}

// esc_multiply(a, b, chunk), local_spgemm.hpp:83-156.
int ref_esc_multiply(int sr, const ref_csr* a, const ref_csr* b, uint64_t chunk, ref_csr* out) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      from_csr(esc_multiply(to_csr<SR>(*a), to_csr<SR>(*b), chunk), out);
      return 0;
    });
  });
}

// naive_multiply(a, b), local_spgemm.hpp:162-210.
int ref_naive_multiply(int sr, const ref_csr* a, const ref_csr* b, ref_csr* out) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      from_csr(naive_multiply(to_csr<SR>(*a), to_csr<SR>(*b)), out);
      return 0;
    });
  });
}

// coo_to_csc then csc_to_csr (formats.hpp:137-180, :291-316): normalised CSR.
int ref_coo_to_csr(int sr, const ref_coo* m, ref_csr* out) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      from_csr(csc_to_csr(coo_to_csc(to_coo<SR>(*m))), out);
      return 0;
    });
  });
}

// coo_to_csc (formats.hpp:137-180).
int ref_coo_to_csc(int sr, const ref_coo* m, ref_csr* out) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      from_csc(coo_to_csc(to_coo<SR>(*m)), out);
      return 0;
    });
  });
}

// matrix_checksum(CsrMatrix) (checksum.hpp:20-38, :45-47).
int ref_checksum_csr(int sr, const ref_csr* m, uint64_t* out) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      *out = matrix_checksum(to_csr<SR>(*m));
      return 0;
    });
  });
}

// matrix_checksum(CscMatrix).
int ref_checksum_csc(int sr, const ref_csr* m, uint64_t* out) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      *out = matrix_checksum(to_csc<SR>(*m));
      return 0;
    });
  });
}

// csr_row_slice / csr_col_slice, summa.hpp:57-98.
int ref_csr_slice(int sr, const ref_csr* m, int by_rows, int64_t begin, int64_t end, ref_csr* out) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      const auto csr = to_csr<SR>(*m);
      from_csr(by_rows ? csr_row_slice(csr, BlockRange{begin, end})
                       : csr_col_slice(csr, BlockRange{begin, end}),
               out);
      return 0;
    });
  });
}

// merge_partials(parts, block_rows, block_cols), summa.hpp:122-172.
// parts[i] are CSR of C^T partials; output is the CSC C block.
int ref_merge_partials(int sr, int nparts, const ref_csr* parts, const int* stages,
                       const int* rounds, int64_t block_rows, int64_t block_cols, ref_csr* out) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      std::vector<Partial<SR>> ps;
      for (int i = 0; i < nparts; ++i) ps.push_back({stages[i], rounds[i], to_csr<SR>(parts[i])});
      from_csc(merge_partials<SR>(std::move(ps), block_rows, block_cols), out);
      return 0;
    });
  });
}

// block_range(n, q, idx), dist_matrix.hpp:23-28; round_range, summa.hpp:103-107.
void ref_block_range(int64_t n, int q, int idx, int64_t* begin, int64_t* end) {
  const BlockRange r = block_range(n, q, idx);
  *begin = r.begin;
  *end = r.end;
}
void ref_round_range(int64_t n, int rounds, int round, int64_t* begin, int64_t* end) {
  const BlockRange r = round_range(n, rounds, round);
  *begin = r.begin;
  *end = r.end;
}

// csc_to_dcsc then dcsc_decompress round trip (formats.hpp:199-250); returns
// the number of nonempty columns (jc size) in *jc_len.
int ref_dcsc_roundtrip(int sr, const ref_csr* csc, int64_t* jc_len, ref_csr* out) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      const auto d = csc_to_dcsc(to_csc<SR>(*csc));
      *jc_len = static_cast<int64_t>(d.jc.size());
      from_csc(dcsc_decompress(d), out);
      return 0;
    });
  });
}

// distribute (dist_matrix.hpp:69-111) on a p-rank square grid: rank's block
// as CSC (dcsc_decompress'ed when stored DCSC), its DCSC flag and extents.
int ref_distribute_block(int sr, const ref_coo* m, int p, int rank, ref_csr* out, int* is_dcsc,
                         int64_t* extents) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      const auto dm = distribute(to_coo<SR>(*m), ProcessGrid{p});
      const auto& blk = dm.blocks.at(static_cast<std::size_t>(rank));
      *is_dcsc = std::holds_alternative<DcscMatrix<SR>>(blk.storage) ? 1 : 0;
      extents[0] = blk.rows.begin;
      extents[1] = blk.rows.end;
      extents[2] = blk.cols.begin;
      extents[3] = blk.cols.end;
      if (*is_dcsc) from_csc(dcsc_decompress(std::get<DcscMatrix<SR>>(blk.storage)), out);
      else from_csc(std::get<CscMatrix<SR>>(blk.storage), out);
      return 0;
    });
  });
}

// summa25_multiply(distribute(A, p), distribute(B, p), bundled model, cfg, opts)
// then gather (summa.hpp:248-349, dist_matrix.hpp:69-141).  ledger receives
// {host_bcasts, device_bcasts, bytes_host, bytes_device, size_exchanges,
//  local_multiply_calls, skipped_stages, peak_bcast_buffer_bytes,
//  sim_comm_seconds, wall_local_multiply, wall_merge, wall_prepare}.
int ref_summa(int sr, const ref_coo* a, const ref_coo* b, int p, int two_round, int mode,
              uint64_t threshold, uint64_t chunk, ref_coo* out, uint64_t* checksum,
              double* ledger) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      const ProcessGrid grid(p);
      const auto da = distribute(to_coo<SR>(*a), grid);
      const auto db = distribute(to_coo<SR>(*b), grid);
      CommConfig cfg;
      cfg.mode = mode == 0 ? CommMode::host_only : mode == 1 ? CommMode::device_only : CommMode::hybrid;
      cfg.threshold_bytes = threshold;
      SummaOptions opts;
      opts.two_round = two_round != 0;
      opts.chunk_nnz = chunk;
      auto res = summa25_multiply(da, db, LatencyModel::bundled_default(), cfg, opts);
      const auto c = gather(res.product);
      if (checksum) *checksum = matrix_checksum(c);
      if (out) from_coo(c, out);
      if (ledger) {
        const auto& l = res.ledger;
        ledger[0] = double(l.host_bcasts);
        ledger[1] = double(l.device_bcasts);
        ledger[2] = double(l.bytes_host_path);
        ledger[3] = double(l.bytes_device_path);
        ledger[4] = double(l.size_exchanges);
        ledger[5] = double(l.local_multiply_calls);
        ledger[6] = double(l.skipped_stages);
        ledger[7] = double(l.peak_bcast_buffer_bytes);
        ledger[8] = l.sim_comm_seconds();
        ledger[9] = l.wall_at(Phase::local_multiply);
        ledger[10] = l.wall_at(Phase::merge);
        ledger[11] = l.wall_at(Phase::prepare);
      }
      return 0;
    });
  });
}

// find_crossover(bundled_default, fanout, lo, hi), tuner.hpp:17-39.
// Returns 1 and writes *out when a crossover exists, else 0.
int ref_find_crossover_bundled(int fanout, uint64_t lo, uint64_t hi, uint64_t* out) {
  const auto r = find_crossover(LatencyModel::bundled_default(), fanout, lo, hi);
  if (!r) return 0;
  *out = *r;
  return 1;
}

// find_crossover on a model FILE (LatencyModel::load_file, latency_model.hpp:
// 169-179): the reference's own tuner consuming curves measured on the box.
// Returns 1 and writes *out on a crossover, 0 without one, -1 on error.
int ref_find_crossover_file(const char* path, int fanout, uint64_t lo, uint64_t hi, uint64_t* out) {
  try {
    const auto m = LatencyModel::load_file(path);
    const auto r = find_crossover(m, fanout, lo, hi);
    if (!r) return 0;
    *out = *r;
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Bundled model path costs (latency_model.hpp:104-109) for the sweep tests.
double ref_bundled_host_total(uint64_t bytes, int fanout) {
  return LatencyModel::bundled_default().host_path_total(bytes, fanout);
}
double ref_bundled_device_total(uint64_t bytes, int fanout) {
  return LatencyModel::bundled_default().device_path_total(bytes, fanout);
}

// CPU baseline: the reference esc_multiply run concurrently by `nthreads`
// threads on disjoint row slices [row_lo, row_hi) of A (it is pure and
// reentrant), each slice times B.  Slicing is outside the
// timed region.  Returns wall seconds of the concurrent multiplies and the
// total output nnz / products.
int ref_esc_rows_mt(int sr, const ref_csr* a, const ref_csr* b, int64_t row_lo, int64_t row_hi,
                    int nthreads, double* seconds, int64_t* nnz_out, int64_t* flops_out,
                    uint64_t* checksum_sum) {
  return guarded([&] {
    return with_ref_sr(sr, [&](auto t) {
      using SR = typename decltype(t)::type;
      const auto A = to_csr<SR>(*a);
      const auto B = to_csr<SR>(*b);
      const int T = std::max(1, nthreads);
      // Balance the slices by product count.
      std::vector<int64_t> prod_prefix(static_cast<std::size_t>(row_hi - row_lo) + 1, 0);
      for (int64_t i = row_lo; i < row_hi; ++i) {
        int64_t f = 0;
        for (int64_t u = A.rowptr[i]; u < A.rowptr[i + 1]; ++u) {
          const int64_t k = A.colids[u];
          f += B.rowptr[k + 1] - B.rowptr[k];
        }
        prod_prefix[i - row_lo + 1] = prod_prefix[i - row_lo] + f;
      }
      const int64_t total = prod_prefix.back();
      std::vector<CsrMatrix<SR>> slices;
      int64_t cut = row_lo;
      for (int w = 0; w < T; ++w) {
        const int64_t target = total * (w + 1) / T;
        int64_t hi = cut;
        while (hi < row_hi && prod_prefix[hi - row_lo] < target) ++hi;
        if (w == T - 1) hi = row_hi;
        slices.push_back(csr_row_slice(A, BlockRange{cut, hi}));
        cut = hi;
      }
      std::vector<CsrMatrix<SR>> outs(slices.size());
      const auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> ts;
      for (std::size_t w = 0; w < slices.size(); ++w) {
        ts.emplace_back([&, w] { outs[w] = esc_multiply(slices[w], B); });
      }
      for (auto& th : ts) th.join();
      const auto t1 = std::chrono::steady_clock::now();
      *seconds = std::chrono::duration<double>(t1 - t0).count();
      int64_t nnz = 0;
      uint64_t sum = 0;
      for (const auto& o : outs) {
        nnz += o.nnz();
        if (checksum_sum) sum += matrix_checksum(o);
      }
      *nnz_out = nnz;
      *flops_out = total;
      if (checksum_sum) *checksum_sum = sum;
      return 0;
    });
  });
}

}  // extern "C"
