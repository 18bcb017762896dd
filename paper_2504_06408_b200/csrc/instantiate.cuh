// Per-semiring instantiation of the device pipeline.  Each built-in semiring
// gets its own translation unit (sr_*.cu) containing one SPG_INSTANTIATE; a
// user-defined semiring is added the same way from the user's own .cu file
// (compiled into the user's shared library against these headers) and
// registered at run time with spg_register_semiring(), which returns the id
// every C-ABI entry point then accepts — the analogue of instantiating the
// reference's templates with a new SemiringLike type (semiring.hpp:28-40).
// tests/custom_sr/maxmin_sr.cu is a complete example.
#pragma once
#include <type_traits>

#include "rows_driver.cuh"

namespace spg {

SPG_HD uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// checksum.hpp:25-33: FNV-1a over the ValueCodec bytes, mixed with the
// coordinates.
template <class V>
SPG_HD uint64_t tuple_hash(int64_t row, int64_t col, const V& v) {
  const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
  uint64_t fh = 0xcbf29ce484222325ULL;
#pragma unroll
  for (int k = 0; k < (int)sizeof(V); ++k) fh = (fh ^ b[k]) * 0x100000001b3ULL;
  uint64_t h = splitmix64((uint64_t)row);
  h ^= splitmix64((uint64_t)col + 0x9e3779b97f4a7c15ULL);
  h ^= fh;
  return splitmix64(h);
}

// tuple_hash with the segment's coordinate hashed once: `seg_h` is
// splitmix64(row) (CSR segment) or splitmix64(col + golden) (CSC segment).
template <class V>
SPG_HD uint64_t tuple_hash_seg(uint64_t seg_h, int64_t other, bool is_csc, const V& v) {
  const uint8_t* b = reinterpret_cast<const uint8_t*>(&v);
  uint64_t fh = 0xcbf29ce484222325ULL;
#pragma unroll
  for (int k = 0; k < (int)sizeof(V); ++k) fh = (fh ^ b[k]) * 0x100000001b3ULL;
  const uint64_t oh = is_csc ? splitmix64((uint64_t)other) : splitmix64((uint64_t)other + 0x9e3779b97f4a7c15ULL);
  return splitmix64(seg_h ^ oh ^ fh);
}

// K8: order-free content checksum, warp per segment, one atomic per CTA.
template <class V>
__global__ void __launch_bounds__(256) checksum_kernel(int64_t nseg, const int64_t* __restrict__ ptr,
                                                       const int32_t* __restrict__ idx,
                                                       const V* __restrict__ vals, int is_csc,
                                                       int64_t row_off, int64_t col_off,
                                                       unsigned long long* out) {
  __shared__ unsigned long long part[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long acc = 0;
  for (int64_t s = warp; s < nseg; s += nwarps) {
    const int64_t b = ptr[s], e = ptr[s + 1];
    if (b == e) continue;
    const uint64_t seg_h = is_csc ? splitmix64((uint64_t)(s + col_off) + 0x9e3779b97f4a7c15ULL)
                                  : splitmix64((uint64_t)(s + row_off));
    const int64_t ooff = is_csc ? row_off : col_off;
    for (int64_t t = b + lane; t < e; t += 32) acc += tuple_hash_seg(seg_h, idx[t] + ooff, is_csc != 0, vals[t]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) part[wid] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += part[w];
    atomicAdd(out, s);
  }
}

constexpr int kSrOpsAbi = 2;  // layout version of SrOps (checked at registration)

struct SrOps {
  int abi;
  int id;  // built-ins: their SPG_SR_* id; user semirings: -1 (the registry assigns one)
  const char* name;
  int value_size;
  bool commutative;
  void (*local_multiply)(spg_ctx*, const spg_dcsr*, const spg_dcsr*, spg_dcsr*, spg_mult_stats*);
  // parts are CSR with identical dims (rows x cols); output rows x cols
  void (*merge)(spg_ctx*, int, const spg_dcsr*, int64_t, int64_t, spg_dcsr*, spg_mult_stats*);
  // sum of tuple terms with coordinate offsets (no dims seed)
  uint64_t (*checksum_part)(spg_ctx*, const spg_dcsr*, int, int64_t, int64_t);
  // distribute's duplicate fold (formats.hpp:160-170): run u covers sorted
  // positions [heads[u], heads[u+1]) (the last ends at n); its values
  // vin[order[p]] fold left to right with SR::add into vout[u]; keep[u] = the
  // result is not SR::is_zero.
  void (*fold_runs)(spg_ctx*, int64_t nu, const int64_t* heads, int64_t n, const int64_t* order,
                    const void* vin, void* vout, uint8_t* keep);
};

// One thread per run of equal (rank, column, row) keys.
template <class SR>
__global__ void __launch_bounds__(256) fold_runs_kernel(int64_t nu, const int64_t* __restrict__ heads, int64_t n,
                                                        const int64_t* __restrict__ order,
                                                        const typename SR::value_type* __restrict__ vin,
                                                        typename SR::value_type* __restrict__ vout,
                                                        uint8_t* __restrict__ keep) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nu; u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = heads[u], e = u + 1 < nu ? heads[u + 1] : n;
    typename SR::value_type acc = vin[order[b]];
    for (int64_t p = b + 1; p < e; ++p) acc = SR::add(acc, vin[order[p]]);
    vout[u] = acc;
    keep[u] = !SR::is_zero(acc);
  }
}

template <class SR>
struct OpsImpl {
  using V = typename SR::value_type;

  static void local_multiply(spg_ctx* c, const spg_dcsr* a, const spg_dcsr* b, spg_dcsr* out,
                             spg_mult_stats* st) {
    MulSource<SR> src{a->ptr, a->idx, static_cast<const V*>(a->vals),
                      b->ptr, b->idx, static_cast<const V*>(b->vals), a->nrows};
    if (run_rows_pattern<SR>(c, src, b, b->ncols, out, st)) return;
    if (!run_rows_br<SR>(c, src, b, b->ncols, out, st)) run_rows<SR>(c, src, b->ncols, out, st, b);
  }

  static void merge(spg_ctx* c, int nparts, const spg_dcsr* parts, int64_t rows, int64_t cols,
                    spg_dcsr* out, spg_mult_stats* st) {
    if (nparts > kMaxMergeParts) fail(SPG_ERR_ARG, "merge: too many partials");
    MergeSource<SR> src{};
    src.nparts = nparts;
    src.nrows = rows;
    for (int q = 0; q < nparts; ++q) {
      src.p.ptr[q] = parts[q].ptr;
      src.p.idx[q] = parts[q].idx;
      src.p.val[q] = parts[q].vals;
    }
    run_rows<SR>(c, src, cols, out, st);
  }

  static uint64_t checksum_part(spg_ctx* c, const spg_dcsr* m, int is_csc, int64_t row_off, int64_t col_off) {
    const int64_t nseg = is_csc ? m->ncols : m->nrows;
    DBuf<unsigned long long> acc(c, 1);
    SPG_CUDA(cudaMemsetAsync(acc.p, 0, sizeof(unsigned long long), c->stream));
    if (nseg > 0 && m->nnz > 0) {
      const int grid = grid_for(c, nseg, 8, 8);
      checksum_kernel<V><<<grid, 256, 0, c->stream>>>(nseg, m->ptr, m->idx, static_cast<const V*>(m->vals),
                                                      is_csc, row_off, col_off, acc.p);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    return d2h_scalar(c, acc.p);
  }

  static void fold_runs(spg_ctx* c, int64_t nu, const int64_t* heads, int64_t n, const int64_t* order,
                        const void* vin, void* vout, uint8_t* keep) {
    if (nu <= 0) return;
    fold_runs_kernel<SR><<<grid_for(c, nu, 256, 8), 256, 0, c->stream>>>(
        nu, heads, n, order, static_cast<const V*>(vin), static_cast<V*>(vout), keep);
    SPG_LAUNCH_CHECK();
    ++c->launches;
  }
};

template <class SR, class = void>
struct sr_has_id : std::false_type {};
template <class SR>
struct sr_has_id<SR, decltype((void)SR::id, void())> : std::true_type {};
template <class SR>
constexpr int sr_id() {
  if constexpr (sr_has_id<SR>::value) return SR::id;
  else return -1;
}

template <class SR>
const SrOps* ops_instance() {
  static const SrOps o{kSrOpsAbi, sr_id<SR>(), SR::name, (int)sizeof(typename SR::value_type), SR::is_commutative_mul,
                       &OpsImpl<SR>::local_multiply, &OpsImpl<SR>::merge, &OpsImpl<SR>::checksum_part,
                       &OpsImpl<SR>::fold_runs};
  return &o;
}

}  // namespace spg

#define SPG_INSTANTIATE(SR, FN) \
  extern "C" __attribute__((visibility("default"))) const spg::SrOps* FN() { return spg::ops_instance<SR>(); }
