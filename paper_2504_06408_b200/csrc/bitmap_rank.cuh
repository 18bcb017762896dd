// Bitmap-rank pipeline for the long rows of a local multiply
// (esc_multiply replacement, local_spgemm.hpp:83-156) — output written
// straight into C, no scratch and no compaction.
//
//   S  br_symbolic_kernel : CTA per row; the row's presence bitmap over ALL
//                           output columns lives in shared memory (one bit per
//                           column: 32 KB for 262 144 columns), every product
//                           column sets its bit (one pass, cols only, no
//                           column panels); nnz_i = popcount.  The bitmap is
//                           streamed to HBM (one slot per row) together with
//                           the columns where the row's rank WINDOWS start
//                           (window k = output ranks [k*capv, (k+1)*capv)).
//   P  exclusive scan of nnz_i -> rowptr of C; C allocated exactly once; the
//      (row, window) work list is expanded from the window counts.
//   N  br_numeric_kernel  : CTA per (row, window) work item; the window's
//                           bitmap words come back into shared memory, a block
//                           scan of their popcounts gives every output column
//                           its RANK = its position in the output row.  Columns
//                           are expanded from the bitmap (sorted without
//                           sorting) and stored contiguously; the products of
//                           the segment slices that fall in the window (binary
//                           search per segment when the row has several
//                           windows) fold with native shared-memory atomics
//                           into acc[rank], which is then copied out as the
//                           window's values.
//
// Item enumeration (br_items): a warp walks its equal share of the row's
// products 32 at a time; the segment of each lane comes from ONE warp-wide
// OR-reduction (REDUX) of the segment starts that fall inside the batch and a
// popcount — no per-lane search and no shuffles — over a per-batch cache of
// the non-empty segments (start, exclusive product prefix, left scalar).
//
// Zero dropping (formats.hpp:129, local_spgemm.hpp:57-58): the symbolic pass
// marks every product column, so an entry whose fold is the semiring zero
// (a zero product, or fp64 cancellation) is written as zero() and counted; the
// rare call that produced any is compacted afterwards (drop_zero_entries).
#pragma once
#include <cub/block/block_reduce.cuh>

#include <type_traits>

#include "accumulate.cuh"

namespace spg {

constexpr int64_t kBrMaxCols = 1 << 19;
constexpr int kBrMaxPanels = 256;  // fine column panels per row (window boundaries fall on them)

// SPG_BR_PROF builds: per-phase cycle totals (thread 0 of every CTA), printed
// by the driver — numeric 0 grab, 1 bitmap in, 2 count pass, 3 rank/emit
// pass, 4 columns out, 5 segment cache, 6 fold, 7 values out; symbolic 8
// grab, 9 segment cache, 10 walk, 11 tail.
#ifdef SPG_BR_PROF
static __device__ unsigned long long br_prof[16];
#define BR_T(k)                                                        \
  if (threadIdx.x == 0) {                                              \
    const long long t_ = clock64();                                    \
    atomicAdd(&br_prof[(k)], (unsigned long long)(t_ - br_t_last));    \
    br_t_last = t_;                                                    \
  }
#define BR_T_INIT long long br_t_last = clock64();
#else
#define BR_T(k)
#define BR_T_INIT
#endif  // output width whose bitmap fits shared memory (64 KB)

// words per bitmap slot: a power of two >= 4096 (whole 16-byte quads for every
// thread, whole fine panels)
__host__ __device__ inline int br_words(int64_t ncols) {
  const int64_t w = (ncols + 31) / 32;
  int n = 4096;
  while (n < w) n <<= 1;
  return n;
}

// mbarrier + bulk-copy (TMA) primitives
__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred P1;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n @!P1 bra WAIT_%=;\n}" ::"r"(
          smem_addr(bar)),
      "r"(phase)
      : "memory");
}

// number of right-operand values that are not SR::small (fast-multiply check)
template <class SR>
__global__ void br_count_not_small_kernel(int64_t n, const typename SR::value_type* __restrict__ v,
                                          unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
    c += SR::small(v[u]) ? 0 : 1;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// bulk copy of nw bitmap words [wb, wb + nw) of slot `slot` into bm (one
// thread; completion = the mbarrier's transaction count)
__device__ __forceinline__ void br_bitmap_copy(uint32_t* bm, const uint32_t* gbm, int64_t slot, int nwords, int wb,
                                               int nw, unsigned long long* bar) {
  fence_proxy_async();  // earlier generic accesses of bm precede the async-proxy writes
  const unsigned bytes = (unsigned)nw * 4u;
  mbar_expect_tx(bar, bytes);
  const char* gsrc = reinterpret_cast<const char*>(gbm + (size_t)slot * nwords + wb);
  for (unsigned o = 0; o < bytes; o += 16384u)
    bulk_g2s(reinterpret_cast<char*>(bm) + o, gsrc + o, min(16384u, bytes - o), bar);
}

// Right operand with column and value interleaved (one 8- or 16-byte load per
// product instead of two): built once per call for values of <= 8 bytes.
template <class V>
struct __align__(sizeof(V) <= 4 ? 8 : 16) BrPack {
  int32_t col;
  V val;
};
template <class V>
__global__ void br_pack_kernel(int64_t nnz, const int32_t* __restrict__ idx, const V* __restrict__ vals,
                               BrPack<V>* __restrict__ out) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nnz; u += (int64_t)gridDim.x * blockDim.x) {
    BrPack<V> p;
    p.col = idx[u];
    p.val = vals[u];
    out[u] = p;
  }
}

// Per-batch cache of the non-empty segments of one row (<= THREADS of them).
template <class V>
struct BrSegs {
  int32_t* b;    // first right-operand entry of the segment slice (nnz(R) < 2^31 on this path)
  int32_t* pre;  // [n + 1] exclusive prefix of the slice lengths
  V* mult;       // left scalar
  static __host__ __device__ size_t bytes(int threads) {
    return ((sizeof(int32_t) * threads + 15) & ~size_t(15)) + ((sizeof(int32_t) * (threads + 1) + 15) & ~size_t(15)) +
           ((sizeof(V) * threads + 15) & ~size_t(15));
  }
  __device__ __forceinline__ void carve(unsigned char* p, int threads) {
    b = reinterpret_cast<int32_t*>(p);
    pre = reinterpret_cast<int32_t*>(p + ((sizeof(int32_t) * threads + 15) & ~size_t(15)));
    mult = reinterpret_cast<V*>(reinterpret_cast<unsigned char*>(pre) +
                                ((sizeof(int32_t) * (threads + 1) + 15) & ~size_t(15)));
  }
};

// One segment per thread, fetched early into registers (its global loads
// then overlap whatever the CTA does before br_seg_build).
template <class V>
struct BrSegReg {
  int64_t b = 0;
  int len = 0;
  V m{};
};
template <class SR, class Src>
__device__ __forceinline__ BrSegReg<typename SR::value_type> br_seg_fetch(const Src& src, int64_t i, int64_t s0, int n) {
  BrSegReg<typename SR::value_type> g;
  g.m = SR::zero();
  if ((int)threadIdx.x < n) {
    int sd;
    src.seg(i, s0 + threadIdx.x, -1, g.b, g.len, sd, g.m);
  }
  return g;
}
// The slice of each segment inside fine panels [p0, p1): the right
// operand's panel offsets poff[k * (npf + 1) + p] (entries of R row k with
// column < p * panel width, computed once per call) bound it — no search.
template <class SR, class Src>
__device__ __forceinline__ BrSegReg<typename SR::value_type> br_seg_fetch_panels(const Src& src,
                                                                                const int32_t* __restrict__ poff,
                                                                                int npf, int p0, int p1, bool restrict_cols,
                                                                                int64_t i, int64_t s0, int n) {
  BrSegReg<typename SR::value_type> g;
  g.m = SR::zero();
  if ((int)threadIdx.x < n) {
    const int32_t k = __ldg(src.lidx + s0 + threadIdx.x);
    g.b = __ldg(src.rptr + k);
    g.m = src.lval[s0 + threadIdx.x];
    if (restrict_cols) {
      const int32_t* po = poff + (int64_t)k * (npf + 1);
      const int32_t a = __ldg(po + p0), e = __ldg(po + p1);
      g.b += a;
      g.len = e - a;
    } else {
      g.len = (int)(__ldg(src.rptr + k + 1) - g.b);
    }
  }
  return g;
}

// Builds the compacted cache from the fetched segments to output columns [clo, chi) when
// `restrict_cols`, drops the empty ones and builds the compacted cache;
// returns the number kept.  Block-wide (ends with a barrier).
template <class SR, class Src, int THREADS, class Scan64>
__device__ __forceinline__ int br_seg_build(const Src& src, const BrSegs<typename SR::value_type>& cs,
                                            const BrSegReg<typename SR::value_type>& g,
                                            typename Scan64::TempStorage& tmp, int* s_cnt, bool* all_small = nullptr) {
  const unsigned long long packed = g.len > 0 ? ((1ull << 32) | (unsigned long long)g.len) : 0ull;
  unsigned long long excl, total;
  Scan64(tmp).ExclusiveSum(packed, excl, total);
  const int nn = (int)(total >> 32);
  if (g.len > 0) {
    const int k = (int)(excl >> 32);
    cs.b[k] = (int32_t)g.b;
    cs.pre[k] = (int)(excl & 0xffffffffull);
    cs.mult[k] = g.m;
  }
  if (threadIdx.x == 0) {
    cs.pre[nn] = (int)(total & 0xffffffffull);
    *s_cnt = 0;
  }
  if constexpr (has_mul_small<SR>::value) {
    const bool ok = __syncthreads_and(g.len == 0 || SR::small(g.m));
    if (all_small) *all_small = ok;
  } else {
    __syncthreads();
    if (all_small) *all_small = false;
  }
  return nn;
}

// Warp `wid` of NW walks its equal share of the cached segments' items,
// 32 * IPL at a time; f(col, value) per item (value = mul(left, right), or
// unset when !kVals).
template <class SR, class Src, int NW, int IPL, bool kVals, bool kPacked, bool kFast = false, class F>
__device__ __forceinline__ void br_items(const Src& src, const BrPack<typename SR::value_type>* __restrict__ pack,
                                         const BrSegs<typename SR::value_type>& cs, int n, int wid, F&& f) {
  using V = typename SR::value_type;
  const int lane = threadIdx.x & 31;
  const int P = cs.pre[n];
  const int lo_q = (int)((int64_t)P * wid / NW), hi_q = (int)((int64_t)P * (wid + 1) / NW);
  if (lo_q >= hi_q) return;
  int s = 0, hs = n;  // s = largest t with pre[t] <= q0
  while (hs - s > 1) {
    const int mid = (s + hs) >> 1;
    if (cs.pre[mid] <= lo_q) s = mid;
    else hs = mid;
  }
  for (int q0 = lo_q; q0 < hi_q; q0 += 32 * IPL) {
    int32_t uu[IPL];
    V mm[IPL];
    const int nxt = s + 1 < n ? cs.pre[s + 1] : INT32_MAX;
    if (nxt >= q0 + 32 * IPL) {  // warp-uniform: the whole step lies in segment s (long segments)
      const int32_t bs = cs.b[s] - cs.pre[s];
      V m{};
      if constexpr (kVals) m = cs.mult[s];
#pragma unroll
      for (int k = 0; k < IPL; ++k) {
        uu[k] = bs + (q0 + 32 * k + lane);
        if constexpr (kVals) mm[k] = m;
      }
      if (nxt == q0 + 32 * IPL) ++s;
    } else {
#pragma unroll
      for (int k = 0; k < IPL; ++k) {
        const int qb = q0 + 32 * k;
        const int t = s + 1 + lane;
        const int d = (t < n ? cs.pre[t] : INT32_MAX) - qb;  // >= 1: s is the last segment starting <= qb
        const unsigned mask = __reduce_or_sync(kFull, d < 32 ? (1u << d) : 0u);
        const int sg = s + __popc(mask & ((2u << lane) - 1u));
        uu[k] = cs.b[sg] + (qb + lane - cs.pre[sg]);
        if constexpr (kVals) mm[k] = cs.mult[sg];
        s += __popc(mask);
        if (s + 1 < n && cs.pre[s + 1] == qb + 32) ++s;
      }
    }
    int32_t cc[IPL];
    V xx[IPL];
#pragma unroll
    for (int k = 0; k < IPL; ++k)
      if (q0 + 32 * k + lane < hi_q) {
        if constexpr (kVals && kPacked) {
          const BrPack<V> pk = pack[uu[k]];
          cc[k] = pk.col;
          xx[k] = pk.val;
        } else if constexpr (kVals) {
          cc[k] = src.col(0, uu[k]);
          xx[k] = src.val(0, uu[k]);
        } else {
          cc[k] = src.col(0, uu[k]);
        }
      }
#pragma unroll
    for (int k = 0; k < IPL; ++k)
      if (q0 + 32 * k + lane < hi_q) {
        if constexpr (kVals && kFast) f(cc[k], SR::mul_small(mm[k], xx[k]), std::true_type{});
        else if constexpr (kVals) f(cc[k], src.item(mm[k], xx[k]), std::false_type{});
        else f(cc[k], V{}, std::false_type{});
      }
  }
}

#ifndef SPG_BR_SKIP
#define SPG_BR_SKIP 0  // 1: read the slot first, skip atomics that cannot change it (measured slower: 19.8 vs 19.1 ms)
#endif
#ifndef SPG_BR_EMIT_LIGHT
#define SPG_BR_EMIT_LIGHT 0  // > 0: words with more columns expanded warp-cooperatively (measured slower: 4 -> +1.6 ms, 8 -> +0.7 ms)
#endif
#ifndef SPG_BR_EMIT_FLAT
#define SPG_BR_EMIT_FLAT 0  // 1: one bit loop across a lane's words (measured slower: 21.2 vs 19.0 ms)
#endif
#ifndef SPG_BR_IPL
#define SPG_BR_IPL 4  // numeric: 32-item steps per warp iteration (loads in flight)
#endif
#ifndef SPG_BR_SYM_IPL
#define SPG_BR_SYM_IPL 2
#endif
#ifndef SPG_BR_SYM_MINB
#define SPG_BR_SYM_MINB 3
#endif

template <class SR, class Src, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) br_symbolic_kernel(Src src, const int64_t* __restrict__ rows,
                                                                    int64_t nrows_bin, int nwords, int capv,
                                                                    int wpp, int npf, int wstride,
                                                                    unsigned long long* __restrict__ work,
                                                                    uint32_t* __restrict__ gbm,
                                                                    int2* __restrict__ wlist,
                                                                    int32_t* __restrict__ nwin_out,
                                                                    int64_t* __restrict__ rownnz) {
  using V = typename SR::value_type;
  static_assert(!Src::kMultiSrc, "bitmap-rank: local multiply sources only");
  constexpr int NW = THREADS / 32;
  using Scan = cub::BlockScan<int, THREADS>;
  using Scan64 = cub::BlockScan<unsigned long long, THREADS>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem_raw);
  BrSegs<V> cs;
  cs.carve(smem_raw + sizeof(uint32_t) * (size_t)nwords, THREADS);
  __shared__ union {
    typename Scan::TempStorage scan;
    typename Scan64::TempStorage scan64;
  } tmp;
  __shared__ long long s_row;
  __shared__ int s_cnt;
  __shared__ int s_pc[kBrMaxPanels];
  BR_T_INIT
  uint4* bq = reinterpret_cast<uint4*>(bm);
  const int nq = nwords >> 2;
  for (int q = threadIdx.x; q < nq; q += THREADS) bq[q] = make_uint4(0u, 0u, 0u, 0u);
  const int wpt = nwords / THREADS;  // contiguous words per thread (multiple of 4)
  const int w0 = threadIdx.x * wpt;
  __syncthreads();
  for (;;) {
    if (threadIdx.x == 0) {
      const unsigned long long r = atomicAdd(work, 1ull);
      s_row = r < (unsigned long long)nrows_bin ? (long long)r : -1;
    }
    __syncthreads();
    BR_T(8);
    const long long r = s_row;
    if (r < 0) break;
    const int64_t i = rows[r];
    const int64_t sb = src.seg_begin(i), nseg = src.seg_end(i) - sb;
    for (int64_t c0 = 0; c0 < nseg; c0 += THREADS) {
      const int n = (int)(nseg - c0 < (int64_t)THREADS ? nseg - c0 : (int64_t)THREADS);
      const int nn = br_seg_build<SR, Src, THREADS, Scan64>(src, cs, br_seg_fetch<SR>(src, i, sb + c0, n), tmp.scan64,
                                                             &s_cnt);
      BR_T(9);
      br_items<SR, Src, NW, SPG_BR_SYM_IPL, false, false>(src, nullptr, cs, nn, (int)(threadIdx.x >> 5), [&](int32_t c, const V&, auto) {
        SPG_DCHECK(c >= 0 && (c >> 5) < nwords);
        atomicOr(&bm[c >> 5], 1u << (c & 31));
      });
      __syncthreads();
      BR_T(10);
    }
    // nnz, outputs per fine panel (wpp words), rank windows = greedy runs of
    // whole panels holding <= capv outputs, bitmap out
    int cnt = 0;
    for (int k = 0; k < wpt; k += 4) {
      const uint4 x = bq[(w0 + k) >> 2];
      cnt += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
    }
    {
      const int tpp = wpp / wpt;  // threads per panel (a power of two <= 32)
      int pc = cnt;
      for (int o = 1; o < tpp; o <<= 1) pc += __shfl_xor_sync(kFull, pc, o);
      if ((threadIdx.x & (tpp - 1)) == 0 && threadIdx.x / tpp < npf) s_pc[threadIdx.x / tpp] = pc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int nwin = 0, run = 0, acc = 0;
      for (int p = 0; p < npf; ++p) {
        const int c = s_pc[p];
        if (p == 0 || acc + c > capv) {
          wlist[r * wstride + nwin++] = make_int2(p, run);
          acc = 0;
        }
        acc += c;
        run += c;
      }
      wlist[r * wstride + nwin] = make_int2(npf, run);
      nwin_out[r] = run > 0 ? nwin : 0;
      rownnz[i] = run;
    }
    uint4* gq = reinterpret_cast<uint4*>(gbm + (size_t)r * nwords);
    for (int q = threadIdx.x; q < nq; q += THREADS) {
      __stcs(gq + q, bq[q]);  // streamed: keeps the right operand resident in L2
      bq[q] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
    BR_T(11);
  }
}

static __global__ void widen_kernel(const int32_t* __restrict__ a, int64_t n, int64_t* __restrict__ b) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= n; k += (int64_t)gridDim.x * blockDim.x)
    b[k] = k < n ? a[k] : 0;
}

// (slot, window) work items, slots in the bitmap bin's (F-descending) order
static __global__ void br_expand_items_kernel(int64_t nslots, const int32_t* __restrict__ nwin,
                                       const int64_t* __restrict__ off, int2* __restrict__ items) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nslots; s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = off[s];
    for (int k = 0; k < nwin[s]; ++k) items[o + k] = make_int2((int)s, k);
  }
}

// n 32-bit words from shared memory (16-byte aligned, readable up to 3 words
// past n) to dst[d ..) at any alignment: 16-byte stores for the aligned body.
__device__ __forceinline__ void smem_words_out(uint32_t* __restrict__ dst, int64_t d, const uint32_t* s, int n,
                                               int tid, int nt) {
  const int head = (int)std::min<int64_t>((4 - (d & 3)) & 3, n);
  if (tid < head) dst[d + tid] = s[tid];
  const int rest = n - head;
  if (rest <= 0) return;
  const int nq = rest >> 2;
  const int sh = head;
  const uint4* sq = reinterpret_cast<const uint4*>(s);
  uint4* dq = reinterpret_cast<uint4*>(dst + d + head);
  for (int k = tid; k < nq; k += nt) {
    const uint4 a = sq[k];
    uint4 o = a;
    if (sh) {
      const uint4 b = sq[k + 1];
      if (sh == 1) o = make_uint4(a.y, a.z, a.w, b.x);
      else if (sh == 2) o = make_uint4(a.z, a.w, b.x, b.y);
      else o = make_uint4(a.w, b.x, b.y, b.z);
    }
    dq[k] = o;
  }
  const int t0 = head + (nq << 2);
  if (tid < n - t0) dst[d + t0 + tid] = s[t0 + tid];
}

template <class V>
__device__ __forceinline__ void smem_values_out(V* __restrict__ dst, int64_t d, const V* s, int n, int tid, int nt) {
  if constexpr (sizeof(V) % 4 == 0) {
    constexpr int WPE = (int)(sizeof(V) / 4);
    smem_words_out(reinterpret_cast<uint32_t*>(dst), d * WPE, reinterpret_cast<const uint32_t*>(s), n * WPE, tid, nt);
  } else {
    for (int e = tid; e < n; e += nt) dst[d + e] = s[e];
  }
}

// shared-memory layout of the numeric kernel
template <class V>
struct BrNumLayout {
  int nw;    // bitmap words held (window words + alignment)
  int capv;  // accumulator entries
  __host__ __device__ size_t off_pre() const { return sizeof(uint32_t) * (size_t)nw; }
  __host__ __device__ size_t off_acc() const {
    return (off_pre() + sizeof(uint16_t) * (size_t)nw + 15) & ~size_t(15);
  }
  __host__ __device__ size_t off_segs() const {
    const size_t acc = std::max(sizeof(V) * (size_t)capv, sizeof(uint32_t) * (size_t)capv * (sizeof(V) >= 4 ? 1 : 0));
    return (off_acc() + acc + 16 + 15) & ~size_t(15);
  }
  __host__ __device__ size_t bytes(int threads) const { return off_segs() + BrSegs<V>::bytes(threads) + 16; }
};

template <class SR, class Src, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) br_numeric_kernel(
    Src src, const BrPack<typename SR::value_type>* __restrict__ pack, const int2* __restrict__ items, int64_t nitems, const int64_t* __restrict__ rows, int64_t ncols,
    int nwords, int capv, int wpp, int npf, int wstride, const int2* __restrict__ wlist,
    const int32_t* __restrict__ poff, bool r_small, unsigned long long* __restrict__ work,
    const uint32_t* __restrict__ gbm, const int64_t* __restrict__ rowptr, int32_t* __restrict__ ccols,
    typename SR::value_type* __restrict__ cvals, unsigned long long* __restrict__ zeros,
    unsigned long long* __restrict__ rowzero) {
  using V = typename SR::value_type;
  static_assert(!Src::kMultiSrc, "bitmap-rank: local multiply sources only");
  constexpr int NW = THREADS / 32;
  using Scan = cub::BlockScan<int, THREADS>;
  using Scan64 = cub::BlockScan<unsigned long long, THREADS>;
  using Red = cub::BlockReduce<int, THREADS>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const BrNumLayout<V> lay{nwords + 8, capv};
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem_raw);
  uint16_t* pre16 = reinterpret_cast<uint16_t*>(smem_raw + lay.off_pre());
  V* acc = reinterpret_cast<V*>(smem_raw + lay.off_acc());
  uint32_t* stage = reinterpret_cast<uint32_t*>(acc);  // column staging (aliases acc)
  BrSegs<V> cs;
  cs.carve(smem_raw + lay.off_segs(), THREADS);
  __shared__ union {
    typename Scan::TempStorage scan;
    typename Scan64::TempStorage scan64;
    typename Red::TempStorage red;
  } tmp;
  __shared__ long long s_item, s_next;
  __shared__ int s_wsum[NW];
  __shared__ int s_cnt;
  __shared__ __align__(8) unsigned long long s_bar;  // bitmap bulk copy completion
  __shared__ bool s_issued;                          // this item's copy was issued ahead
  __shared__ bool s_zero_seen;                       // a zero product was skipped in this item
  BR_T_INIT
  if (threadIdx.x == 0) {
    s_issued = false;
    const unsigned long long w = atomicAdd(work, 1ull);
    s_next = w < (unsigned long long)nitems ? (long long)w : -1;
    mbar_init(&s_bar, 1);
    fence_mbar_init();
  }
  unsigned phase = 0;
  for (;;) {
    // work items are grabbed one ahead: the next item's bitmap words are
    // prefetched into L2 while this one is processed
    if (threadIdx.x == 0) {
      s_item = s_next;
      s_zero_seen = false;
      long long nx = -1;
      if (s_next >= 0) {
        const unsigned long long w = atomicAdd(work, 1ull);
        nx = w < (unsigned long long)nitems ? (long long)w : -1;
      }
      s_next = nx;
    }
    __syncthreads();
    BR_T(0);
    const long long wi = s_item;
    if (wi < 0) break;
    const int2 it = items[wi];
    const int64_t slot = it.x;
    const int k = it.y;
    const int64_t i = rows[slot];
    const int2 w0 = wlist[slot * wstride + k], w1 = wlist[slot * wstride + k + 1];
    const int p0 = w0.x, p1 = w1.x;                      // fine panels [p0, p1)
    const int r0 = w0.y, nr = w1.y - w0.y;               // output ranks [r0, r0 + nr)
    const int wb = p0 * wpp, nw = (p1 - p0) * wpp;       // bitmap words held
    SPG_DCHECK(p0 >= 0 && p0 < p1 && p1 <= npf && nr >= 0 && nr <= capv && wb + nw <= nwords);
    // 1. the window's bitmap words: one bulk (TMA) copy into shared memory,
    //    completing on an mbarrier (issued at the end of the previous item's
    //    fold when this item was known then; else now)
    if (threadIdx.x == 0 && !s_issued) br_bitmap_copy(bm, gbm, slot, nwords, wb, nw, &s_bar);
    // this item's segments (slices of the window's panels): loads issued now
    const int64_t sb = src.seg_begin(i), nseg = src.seg_end(i) - sb;
    const bool restrict_cols = p0 > 0 || p1 < npf;
    const BrSegReg<V> g0 =
        br_seg_fetch_panels<SR>(src, poff, npf, p0, p1, restrict_cols, i, sb, (int)(nseg < THREADS ? nseg : THREADS));
    const int64_t base = rowptr[i];
    mbar_wait(&s_bar, phase);
    phase ^= 1u;
    BR_T(1);
    // 2. ranks: lane t of the CTA owns L consecutive words (L a power of two),
    //    visited in an order rotated by its bank group so the lanes of a warp
    //    hit distinct banks; pass 1 masks + counts, one scan of the lanes'
    //    counts, pass 2 stores each word's first rank and emits its columns in
    //    rank order into the stage (stored contiguously after a barrier)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int L = 1;
    while (L * THREADS < nw) L <<= 1;
    const int jt0 = threadIdx.x * L;
    const int rot = L >= 32 ? lane & (L - 1) : (lane / (32 / L)) & (L - 1);
    int tcnt = 0, thi = 0;
    for (int k = 0; k < L; ++k) {
      const int j = jt0 + ((k + rot) & (L - 1));
      if (j < nw) {
        const int c = __popc(bm[j]);
        tcnt += c;
        if (k < L - rot) thi += c;
      }
    }
    int incl = tcnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += t;
    }
    if (lane == 31) s_wsum[wid] = incl;
    __syncthreads();
    BR_T(2);
    {
      int start = incl - tcnt;
      for (int w = 0; w < wid; ++w) start += s_wsum[w];
      int rk = start + (tcnt - thi);  // rank of the first word visited (word rot of the chunk)
      auto put = [&](int r, uint32_t col) {
        if constexpr (sizeof(V) >= 4) stage[r] = col;
        else ccols[base + r0 + r] = col;
      };
#if SPG_BR_EMIT_LIGHT > 0
      // words with <= SPG_BR_EMIT_LIGHT columns: expanded by their lane;
      // denser words: by the whole warp, one bit per lane (no lane waits
      // for another lane's long bit loop)
      for (int k = 0; k < L; ++k) {
        if (k == L - rot) rk = start;  // wrapped to word 0 of the chunk
        const int j = jt0 + ((k + rot) & (L - 1));
        uint32_t x = 0u;
        if (j < nw) {
          x = bm[j];
          pre16[j] = (uint16_t)rk;
        }
        const uint32_t cb = (uint32_t)(wb + j) << 5;
        const int pc = __popc(x);
        SPG_DCHECK(rk + pc <= nr);
        if (pc <= SPG_BR_EMIT_LIGHT) {
          uint32_t y = x;
#pragma unroll
          for (int u = 0; u < SPG_BR_EMIT_LIGHT; ++u)
            if (y) {
              put(rk + u, cb + __ffs(y) - 1);
              y &= y - 1;
            }
        }
        for (unsigned hm = __ballot_sync(kFull, pc > SPG_BR_EMIT_LIGHT); hm; hm &= hm - 1) {
          const int srcl = __ffs(hm) - 1;
          const uint32_t xh = __shfl_sync(kFull, x, srcl);
          const int rh = __shfl_sync(kFull, rk, srcl);
          const uint32_t cbh = __shfl_sync(kFull, cb, srcl);
          if ((xh >> lane) & 1u) put(rh + __popc(xh & ((1u << lane) - 1u)), cbh + lane);
        }
        rk += pc;
      }
#elif SPG_BR_EMIT_FLAT
      // one loop over all the columns of the lane's L words (a word is
      // entered when the previous one is exhausted): the warp runs
      // max-over-lanes(columns + words) steps instead of, per word,
      // max-over-lanes(columns of that word)
      {
        int k = -1;
        uint32_t y = 0u, cb = 0u;
        for (;;) {
          while (y == 0u && k + 1 < L) {
            ++k;
            if (k == L - rot) rk = start;  // wrapped to word 0 of the chunk
            const int j = jt0 + ((k + rot) & (L - 1));
            if (j < nw) {
              y = bm[j];
              pre16[j] = (uint16_t)rk;
              cb = (uint32_t)(wb + j) << 5;
              SPG_DCHECK(rk + __popc(y) <= nr);
            }
          }
          if (y == 0u) break;
          put(rk++, cb + __ffs(y) - 1);
          y &= y - 1;
        }
      }
#else
      for (int k = 0; k < L; ++k) {
        if (k == L - rot) rk = start;  // wrapped to word 0 of the chunk
        const int j = jt0 + ((k + rot) & (L - 1));
        if (j < nw) {
          const uint32_t x = bm[j];
          pre16[j] = (uint16_t)rk;
          const uint32_t cb = (uint32_t)(wb + j) << 5;
          SPG_DCHECK(rk + __popc(x) <= nr);
          for (uint32_t y = x; y; y &= y - 1) put(rk++, cb + __ffs(y) - 1);
        }
      }
#endif
    }
    __syncthreads();
    BR_T(3);
    if constexpr (sizeof(V) >= 4) {
      smem_words_out(reinterpret_cast<uint32_t*>(ccols), base + r0, stage, nr, threadIdx.x, THREADS);
      __syncthreads();
      BR_T(4);
    }
    for (int e = threadIdx.x; e < nr; e += THREADS) acc[e] = SR::zero();
    // 3. fold the window's products into acc[rank]
    for (int64_t c0 = 0; c0 < nseg; c0 += THREADS) {
      const int n = (int)(nseg - c0 < (int64_t)THREADS ? nseg - c0 : (int64_t)THREADS);
      const BrSegReg<V> g = c0 == 0 ? g0 : br_seg_fetch_panels<SR>(src, poff, npf, p0, p1, restrict_cols, i, sb + c0, n);
      bool small = false;
      const int nn = br_seg_build<SR, Src, THREADS, Scan64>(src, cs, g, tmp.scan64, &s_cnt, &small);
      BR_T(5);
      auto fold = [&](int32_t c, const V& v, auto fast) {
        if constexpr (!decltype(fast)::value) {
          if (SR::is_zero(v)) {  // add(x, zero) == x; its column may end up holding zero()
            s_zero_seen = true;
            return;
          }
        }
        const int j = (c >> 5) - wb;
        SPG_DCHECK(j >= 0 && j < nw);
        const int rk = (int)pre16[j] + __popc(bm[j] & ((1u << (c & 31)) - 1u));
        SPG_DCHECK(rk >= 0 && rk < nr && (bm[j] >> (c & 31) & 1u));  // every product column is in the bitmap
        if constexpr (SPG_BR_SKIP && has_improves<SR>::value) {
          if (!SR::improves(v, *reinterpret_cast<volatile V*>(&acc[rk]))) return;  // cannot lower the slot
        }
        atomic_accumulate<SR, true>(&acc[rk], v);
      };
      constexpr int IPL = sizeof(V) > 4 ? 2 : SPG_BR_IPL;
      if constexpr (has_mul_small<SR>::value && sizeof(V) <= 8) {
        if (small && r_small) br_items<SR, Src, NW, IPL, true, true, true>(src, pack, cs, nn, (int)(threadIdx.x >> 5), fold);
        else br_items<SR, Src, NW, IPL, true, true, false>(src, pack, cs, nn, (int)(threadIdx.x >> 5), fold);
      } else {
        br_items<SR, Src, NW, IPL, true, (sizeof(V) <= 8), false>(src, pack, cs, nn, (int)(threadIdx.x >> 5), fold);
      }
      __syncthreads();
      BR_T(6);
    }
    // the fold is done with bm: start the next item's bitmap copy now so it
    // lands while this item's values go out
    if (threadIdx.x == 0) {
      const long long nx = s_next;
      s_issued = nx >= 0;
      if (nx >= 0) {
        const int2 jt = items[nx];
        const int q0 = wlist[(int64_t)jt.x * wstride + jt.y].x, q1 = wlist[(int64_t)jt.x * wstride + jt.y + 1].x;
        br_bitmap_copy(bm, gbm, jt.x, nwords, q0 * wpp, (q1 - q0) * wpp, &s_bar);
      }
    }
    // 4. values out (zero() entries counted for the drop-zeros fix-up)
    // an entry folds to zero() only if a zero product was skipped or the add
    // can cancel: count such entries only then (drop_zero_entries fix-up)
    if (AddCanCancel<SR>::value || s_zero_seen) {
      int zc = 0;
      for (int e = threadIdx.x; e < nr; e += THREADS) zc += SR::is_zero(acc[e]) ? 1 : 0;
      const int zt = Red(tmp.red).Sum(zc);
      if (threadIdx.x == 0 && zt > 0) {
        atomicAdd(rowzero + i, (unsigned long long)zt);
        atomicAdd(zeros, (unsigned long long)zt);
      }
    }
    smem_values_out<V>(cvals, base + r0, acc, nr, threadIdx.x, THREADS);
    __syncthreads();
    BR_T(7);
  }
}

// ---------------------------------------------------------------------------
// Pattern-only semirings (Boolean): every product of non-zero operands is
// one() and the fold is idempotent, so C is the product's sparsity pattern.
// br_pattern_kernel walks a row's products column-only, one column SUPER-PANEL
// of SP columns at a time (a 64 KB shared-memory bitmap; each segment's slice
// of the super-panel comes from the right operand's panel offsets), so any
// output width works without stored bitmaps:
//   MODE 0: nnz_i = sum of the super-panels' popcounts;
//   MODE 1: (after the rowptr scan) the columns are emitted in order straight
//           into C and the values set to one().
// ---------------------------------------------------------------------------
template <class SR, class Src, int THREADS, int MODE>
__global__ void __launch_bounds__(THREADS, 3) br_pattern_kernel(Src src, const int64_t* __restrict__ rows,
                                                                int64_t nrows_bin, int spw, int nsp,
                                                                const int32_t* __restrict__ poff,
                                                                unsigned long long* __restrict__ work,
                                                                int64_t* __restrict__ rownnz,
                                                                const int64_t* __restrict__ rowptr,
                                                                int32_t* __restrict__ ccols,
                                                                typename SR::value_type* __restrict__ cvals) {
  using V = typename SR::value_type;
  static_assert(!Src::kMultiSrc, "pattern path: local multiply sources only");
  constexpr int NW = THREADS / 32;
  using Scan = cub::BlockScan<int, THREADS>;
  using Scan64 = cub::BlockScan<unsigned long long, THREADS>;
  using Red = cub::BlockReduce<int, THREADS>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem_raw);  // [spw]
  uint32_t* sm = bm + spw;                                // [spw / 32] summary: bit w = word w non-empty
  BrSegs<V> cs;
  cs.carve(smem_raw + sizeof(uint32_t) * ((size_t)spw + spw / 32), THREADS);
  __shared__ union {
    typename Scan::TempStorage scan;
    typename Scan64::TempStorage scan64;
    typename Red::TempStorage red;
  } tmp;
  __shared__ long long s_row;
  __shared__ int s_any;
  __shared__ int s_wcnt[NW];
  const int wpt = spw / THREADS;  // contiguous words per thread (<= 32: inside one summary word)
  const int w0 = threadIdx.x * wpt;
  const uint32_t my_mask = wpt >= 32 ? 0xffffffffu : ((1u << wpt) - 1u) << (w0 & 31);  // my words in sm[w0 >> 5]
  for (int q = threadIdx.x; q < spw; q += THREADS) bm[q] = 0u;
  for (int q = threadIdx.x; q < spw / 32; q += THREADS) sm[q] = 0u;
  __syncthreads();
  for (;;) {
    if (threadIdx.x == 0) {
      const unsigned long long r = atomicAdd(work, 1ull);
      s_row = r < (unsigned long long)nrows_bin ? (long long)r : -1;
    }
    __syncthreads();
    const long long r = s_row;
    if (r < 0) break;
    const int64_t i = rows[r];
    const int64_t sb = src.seg_begin(i), nseg = src.seg_end(i) - sb;
    int64_t run = MODE == 1 ? rowptr[i] : 0;  // next output position (MODE 1) / row count (MODE 0)
    for (int sp = 0; sp < nsp; ++sp) {
      if (threadIdx.x == 0) s_any = 0;
      for (int64_t c0 = 0; c0 < nseg; c0 += THREADS) {
        const int n = (int)(nseg - c0 < (int64_t)THREADS ? nseg - c0 : (int64_t)THREADS);
        int dummy;
        const int nn = br_seg_build<SR, Src, THREADS, Scan64>(
            src, cs, br_seg_fetch_panels<SR>(src, poff, nsp, sp, sp + 1, nsp > 1, i, sb + c0, n), tmp.scan64, &dummy);
        if (nn > 0 && threadIdx.x == 0) s_any = 1;
        const int32_t cbase = sp * spw * 32;
        br_items<SR, Src, NW, 2, false, false>(src, nullptr, cs, nn, (int)(threadIdx.x >> 5),
                                               [&](int32_t c, const V&, auto) {
                                                 const int cc = c - cbase;
                                                 SPG_DCHECK(cc >= 0 && (cc >> 5) < spw);
                                                 atomicOr(&bm[cc >> 5], 1u << (cc & 31));
                                                 atomicOr(&sm[cc >> 10], 1u << ((cc >> 5) & 31));
                                               });
        __syncthreads();
      }
      if (!s_any) continue;  // no products in this super-panel: the bitmap is still clear
      // only the words the summary marks non-empty are read (and cleared):
      // a row's outputs fill ~1 % of a 4 M-column output's words
      const uint32_t mine = sm[w0 >> 5] & my_mask;
      int cnt = 0;
      for (uint32_t y = mine; y; y &= y - 1) cnt += __popc(bm[(w0 & ~31) + __ffs(y) - 1]);
      if constexpr (MODE == 0) {
        run += Red(tmp.red).Sum(cnt);  // valid in thread 0, the only reader
      } else {
        // warp w owns the contiguous words [w * ww, (w + 1) * ww), lanes
        // interleaved; per 32-word group a warp scan, then a flattened
        // emission — lane e of every 32-output step finds its word by a
        // shuffle search — so each store instruction writes 128 contiguous bytes
        (void)cnt;
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        const int ww = spw / NW, wb0 = wid * ww;  // ww <= 1024 words: <= 32 groups of 32 words
        // lane l holds the summary word of the warp's group l; only non-empty
        // groups and, inside them, non-empty words are visited
        const uint32_t swl = lane < (ww >> 5) ? sm[(wb0 >> 5) + lane] : 0u;
        int wc = 0;
        for (uint32_t y = swl; y; y &= y - 1) wc += __popc(bm[wb0 + (lane << 5) + __ffs(y) - 1]);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) wc += __shfl_xor_sync(kFull, wc, d);
        if (lane == 0) s_wcnt[wid] = wc;
        __syncthreads();
        int64_t o = run;
        int tot = 0;
        for (int q = 0; q < NW; ++q) {
          const int v = s_wcnt[q];
          if (q < wid) o += v;
          tot += v;
        }
        const int32_t cb = sp * spw * 32;
        for (unsigned gm = __ballot_sync(kFull, swl != 0u); gm; gm &= gm - 1) {
          const int gl = __ffs(gm) - 1;
          const uint32_t sg = __shfl_sync(kFull, swl, gl);  // the group's 32 words (warp-uniform)
          const int g = gl << 5;
          const uint32_t x = (sg >> lane) & 1u ? bm[wb0 + g + lane] : 0u;
          const int c = __popc(x);
          if (__reduce_max_sync(kFull, (unsigned)c) <= 3u) {
            // sparse group (<= 3 columns per word): a lane's first rank is
            // sum_k popc(ballot(c >= k) below it); each lane writes its own
            const unsigned m1 = __ballot_sync(kFull, c >= 1), m2 = __ballot_sync(kFull, c >= 2),
                           m3 = __ballot_sync(kFull, c >= 3), lt = (1u << lane) - 1u;
            int pos = __popc(m1 & lt) + __popc(m2 & lt) + __popc(m3 & lt);
            const uint32_t wcb = cb + ((uint32_t)(wb0 + g + lane) << 5);
            for (uint32_t y = x; y; y &= y - 1) ccols[o + pos++] = wcb + __ffs(y) - 1;
            o += __popc(m1) + __popc(m2) + __popc(m3);
            continue;
          }
          int incl = c;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const int t = __shfl_up_sync(kFull, incl, d);
            if (lane >= d) incl += t;
          }
          const int total = __shfl_sync(kFull, incl, 31);
          const int excl = incl - c;
          for (int q0 = 0; q0 < total; q0 += 32) {
            const int q = q0 + lane;
            int own = 0;
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1) {
              const int v = __shfl_sync(kFull, incl, own + step - 1);
              if (v <= q) own += step;
            }
            const uint32_t xo = __shfl_sync(kFull, x, own);
            const int eo = __shfl_sync(kFull, excl, own);
            if (q < total) ccols[o + q] = cb + ((wb0 + g + own) << 5) + nth_set_bit(xo, q - eo);
          }
          o += total;
        }
        for (int e = threadIdx.x; e < tot; e += THREADS) cvals[run + e] = SR::one();  // coalesced
        run += tot;
      }
      __syncthreads();  // counts / emission read the bitmap before it is cleared
      for (uint32_t y = mine; y; y &= y - 1) bm[(w0 & ~31) + __ffs(y) - 1] = 0u;
      __syncthreads();  // every thread read its summary bits before they are cleared
      for (int q = threadIdx.x; q < spw / 32; q += THREADS) sm[q] = 0u;
      __syncthreads();
    }
    if constexpr (MODE == 0) {
      if (threadIdx.x == 0) rownnz[i] = run;
    }
    __syncthreads();
  }
}

// non-zero check of operand values (pattern path eligibility)
template <class SR>
__global__ void count_zero_values_kernel(int64_t n, const typename SR::value_type* __restrict__ v,
                                         unsigned long long* __restrict__ out) {
  unsigned long long c = 0;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
    c += SR::is_zero(v[u]) ? 1 : 0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Rare fix-up: drop entries whose value is the semiring zero (warp per row;
// rows without such entries are copied as they are).
template <class SR>
__global__ void __launch_bounds__(256) drop_zero_entries_kernel(int64_t nrows, const int64_t* __restrict__ optr,
                                                                const int32_t* __restrict__ ocols,
                                                                const typename SR::value_type* __restrict__ ovals,
                                                                const int64_t* __restrict__ nptr,
                                                                int32_t* __restrict__ ncols_out,
                                                                typename SR::value_type* __restrict__ nvals) {
  using V = typename SR::value_type;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nrows; i += nwarps) {
    const int64_t b = optr[i], e = optr[i + 1];
    int64_t d = nptr[i];
    for (int64_t t0 = b; t0 < e; t0 += 32) {
      const int64_t t = t0 + lane;
      bool keep = false;
      int32_t c = 0;
      V v{};
      if (t < e) {
        c = ocols[t];
        v = ovals[t];
        keep = !SR::is_zero(v);
      }
      const unsigned m = __ballot_sync(kFull, keep);
      if (keep) {
        const int k = __popc(m & ((1u << lane) - 1u));
        ncols_out[d + k] = c;
        nvals[d + k] = v;
      }
      d += __popc(m);
    }
  }
}

static __global__ void br_kept_counts_kernel(int64_t nrows, const int64_t* __restrict__ optr,
                                      const unsigned long long* __restrict__ rowzero, int64_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x)
    cnt[i] = optr[i + 1] - optr[i] - (int64_t)rowzero[i];
}

}  // namespace spg
