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

#include "accumulate.cuh"

namespace spg {

constexpr int64_t kBrMaxCols = 1 << 19;  // output width whose bitmap fits shared memory (64 KB)

// words per bitmap slot, padded to a multiple of 4096 (16-byte quads for
// every thread of the 512- and 1024-thread kernels)
__host__ __device__ inline int br_words(int64_t ncols) {
  const int64_t w = (ncols + 31) / 32;
  return (int)((w + 4095) / 4096 * 4096);
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

// lower_bound over the sorted columns [lo, hi) of a right-operand row
template <class Src>
__device__ __forceinline__ int64_t br_lower_bound(const Src& src, int64_t lo, int64_t hi, int32_t x) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (src.col(0, mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

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
// Restricts the fetched segments to output columns [clo, chi) when
// `restrict_cols`, drops the empty ones and builds the compacted cache;
// returns the number kept.  Block-wide (ends with a barrier).
template <class SR, class Src, int THREADS, class Scan64>
__device__ __forceinline__ int br_seg_build(const Src& src, const BrSegs<typename SR::value_type>& cs,
                                            BrSegReg<typename SR::value_type> g, int32_t clo, int32_t chi,
                                            bool restrict_cols, typename Scan64::TempStorage& tmp) {
  if (restrict_cols && g.len > 0) {
    const int64_t f = br_lower_bound(src, g.b, g.b + g.len, clo);
    const int64_t e = br_lower_bound(src, f, g.b + g.len, chi);
    g.b = f;
    g.len = (int)(e - f);
  }
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
  if (threadIdx.x == 0) cs.pre[nn] = (int)(total & 0xffffffffull);
  __syncthreads();
  return nn;
}

// Warp `wid` of NW walks its equal share of the cached segments' items,
// 32 * IPL at a time; f(col, value) per item (value = mul(left, right), or
// unset when !kVals).
template <class SR, class Src, int NW, int IPL, bool kVals, bool kPacked, class F>
__device__ __forceinline__ void br_items(const Src& src, const BrPack<typename SR::value_type>* __restrict__ pack,
                                         const BrSegs<typename SR::value_type>& cs, int n, F&& f) {
  using V = typename SR::value_type;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
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
        if constexpr (kVals) f(cc[k], src.item(mm[k], xx[k]));
        else f(cc[k], V{});
      }
  }
}

#ifndef SPG_BR_IPL
#define SPG_BR_IPL 4
#endif

template <class SR, class Src, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) br_symbolic_kernel(Src src, const int64_t* __restrict__ rows,
                                                                    int64_t nrows_bin, int nwords, int capv,
                                                                    int wstride, unsigned long long* __restrict__ work,
                                                                    uint32_t* __restrict__ gbm,
                                                                    int32_t* __restrict__ wcol,
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
    const long long r = s_row;
    if (r < 0) break;
    const int64_t i = rows[r];
    const int64_t sb = src.seg_begin(i), nseg = src.seg_end(i) - sb;
    for (int64_t c0 = 0; c0 < nseg; c0 += THREADS) {
      const int n = (int)(nseg - c0 < (int64_t)THREADS ? nseg - c0 : (int64_t)THREADS);
      const int nn = br_seg_build<SR, Src, THREADS, Scan64>(src, cs, br_seg_fetch<SR>(src, i, sb + c0, n), 0, 0, false,
                                                             tmp.scan64);
      br_items<SR, Src, NW, 2, false, false>(src, nullptr, cs, nn, [&](int32_t c, const V&) {
        atomicOr(&bm[c >> 5], 1u << (c & 31));
      });
      __syncthreads();
    }
    // nnz, window start columns (rank k * capv), bitmap out
    int cnt = 0;
    for (int k = 0; k < wpt; k += 4) {
      const uint4 x = bq[(w0 + k) >> 2];
      cnt += __popc(x.x) + __popc(x.y) + __popc(x.z) + __popc(x.w);
    }
    int pre, total;
    Scan(tmp.scan).ExclusiveSum(cnt, pre, total);
    if (cnt > 0) {
      int k = pre <= 0 ? 1 : (pre + capv - 1) / capv;
      if (k == 0) k = 1;
      int run = pre;
      for (int q = 0; q < wpt && (int64_t)k * capv < pre + cnt; ++q) {
        const uint32_t x = bm[w0 + q];
        const int c = __popc(x);
        while ((int64_t)k * capv < run + c) {
          wcol[r * wstride + k] = ((w0 + q) << 5) + nth_set_bit(x, k * capv - run);
          ++k;
        }
        run += c;
      }
    }
    if (threadIdx.x == 0) {
      wcol[r * wstride] = 0;
      nwin_out[r] = (total + capv - 1) / capv;
      rownnz[i] = total;
    }
    __syncthreads();
    uint4* gq = reinterpret_cast<uint4*>(gbm + (size_t)r * nwords);
    for (int q = threadIdx.x; q < nq; q += THREADS) {
      __stcs(gq + q, bq[q]);  // streamed: keeps the right operand resident in L2
      bq[q] = make_uint4(0u, 0u, 0u, 0u);
    }
    __syncthreads();
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
    int nwords, int capv, int wstride, const int32_t* __restrict__ wcol, unsigned long long* __restrict__ work,
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
  if (threadIdx.x == 0) {
    const unsigned long long w = atomicAdd(work, 1ull);
    s_next = w < (unsigned long long)nitems ? (long long)w : -1;
  }
  for (;;) {
    // work items are grabbed one ahead: the next item's bitmap words are
    // prefetched into L2 while this one is processed
    if (threadIdx.x == 0) {
      s_item = s_next;
      long long nx = -1;
      if (s_next >= 0) {
        const unsigned long long w = atomicAdd(work, 1ull);
        nx = w < (unsigned long long)nitems ? (long long)w : -1;
      }
      s_next = nx;
    }
    __syncthreads();
    const long long wi = s_item;
    if (wi < 0) break;
    const int2 it = items[wi];
    const int64_t slot = it.x;
    const int k = it.y;
    const int64_t i = rows[slot];
    // this item's segments: loads issued now, consumed after the bitmap work
    const int64_t sb = src.seg_begin(i), nseg = src.seg_end(i) - sb;
    const BrSegReg<V> g0 = br_seg_fetch<SR>(src, i, sb, (int)(nseg < THREADS ? nseg : THREADS));
    const int64_t base = rowptr[i];
    const int nnz = (int)(rowptr[i + 1] - base);
    const int nwin = (nnz + capv - 1) / capv;
    const int r0 = k * capv;
    const int nr = min(capv, nnz - r0);
    const int32_t clo = wcol[slot * wstride + k];
    const int32_t chi = k + 1 < nwin ? wcol[slot * wstride + k + 1] : (int32_t)ncols;
    const int wb = (clo >> 5) & ~3;                       // first word held (quad aligned)
    const int nw = ((((chi + 31) >> 5) - wb) + 3) & ~3;  // words held
    {
      const long long nx = s_next;
      if (nx >= 0) {  // L2 prefetch of the next item's bitmap words (128 B lines)
        const int2 jt = items[nx];
        const int64_t nrow = rows[jt.x];
        const int64_t nb0 = rowptr[nrow];
        const int nnz2 = (int)(rowptr[nrow + 1] - nb0);
        const int nwin2 = (nnz2 + capv - 1) / capv;
        const int32_t c0 = wcol[(int64_t)jt.x * wstride + jt.y];
        const int32_t c1 = jt.y + 1 < nwin2 ? wcol[(int64_t)jt.x * wstride + jt.y + 1] : (int32_t)ncols;
        const char* p0 = reinterpret_cast<const char*>(gbm + (size_t)jt.x * nwords + ((c0 >> 5) & ~31));
        const int nl = (((c1 + 31) >> 5) - ((c0 >> 5) & ~31) + 31) >> 5;
        for (int l = threadIdx.x; l < nl; l += THREADS) asm volatile("prefetch.global.L2 [%0];" ::"l"(p0 + 128 * l));
      }
    }
    // 1. the window's bitmap words; bits outside [clo, chi) cleared
    {
      const uint4* gq = reinterpret_cast<const uint4*>(gbm + (size_t)slot * nwords + wb);
      uint4* bq = reinterpret_cast<uint4*>(bm);
      for (int q = threadIdx.x; q < (nw >> 2); q += THREADS) bq[q] = __ldcs(gq + q);
    }
    __syncthreads();
    // 2. ranks: warp w owns the contiguous words [w*per, (w+1)*per), lanes
    //    interleaved (conflict-free); pass 1 masks + counts, pass 2 scans per
    //    32 words, stores the word's first rank and emits its columns in rank
    //    order into the stage (stored contiguously after a barrier)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int per = ((nw + NW * 32 - 1) / (NW * 32)) * 32;
    const int jw0 = wid * per, jw1 = min(nw, jw0 + per);
    {
      int cnt = 0;
      for (int j = jw0 + lane; j < jw1; j += 32) {
        const int c0 = (wb + j) << 5;
        uint32_t x = bm[j];
        if (c0 < clo || c0 + 32 > chi) {
          if (c0 < clo) x = clo - c0 >= 32 ? 0u : x & ~((1u << (clo - c0)) - 1u);
          if (c0 + 32 > chi) x = chi <= c0 ? 0u : x & ((1u << (chi - c0)) - 1u);
          bm[j] = x;
        }
        cnt += __popc(x);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
      if (lane == 0) s_wsum[wid] = cnt;
    }
    __syncthreads();
    {
      int run = 0;
      for (int w = 0; w < wid; ++w) run += s_wsum[w];
      for (int j = jw0 + lane; j - lane < jw1; j += 32) {
        const uint32_t x = j < jw1 ? bm[j] : 0u;
        const int c = __popc(x);
        int incl = c;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
          const int t = __shfl_up_sync(kFull, incl, d);
          if (lane >= d) incl += t;
        }
        int rk = run + incl - c;
        if (j < jw1) pre16[j] = (uint16_t)rk;
        const uint32_t cb = (uint32_t)(wb + j) << 5;
        if constexpr (sizeof(V) >= 4) {
          for (uint32_t y = x; y; y &= y - 1) stage[rk++] = cb + __ffs(y) - 1;
        } else {
          for (uint32_t y = x; y; y &= y - 1) ccols[base + r0 + rk++] = cb + __ffs(y) - 1;
        }
        run += __shfl_sync(kFull, incl, 31);
      }
    }
    __syncthreads();
    if constexpr (sizeof(V) >= 4) {
      smem_words_out(reinterpret_cast<uint32_t*>(ccols), base + r0, stage, nr, threadIdx.x, THREADS);
      __syncthreads();
    }
    for (int e = threadIdx.x; e < nr; e += THREADS) acc[e] = SR::zero();
    // 3. fold the window's products into acc[rank]
    for (int64_t c0 = 0; c0 < nseg; c0 += THREADS) {
      const int n = (int)(nseg - c0 < (int64_t)THREADS ? nseg - c0 : (int64_t)THREADS);
      const BrSegReg<V> g = c0 == 0 ? g0 : br_seg_fetch<SR>(src, i, sb + c0, n);
      const int nn = br_seg_build<SR, Src, THREADS, Scan64>(src, cs, g, clo, chi, nwin > 1, tmp.scan64);
      br_items<SR, Src, NW, (sizeof(V) > 4 ? 2 : SPG_BR_IPL), true, (sizeof(V) <= 8)>(src, pack, cs, nn,
                                                                                      [&](int32_t c, const V& v) {
        if (SR::is_zero(v)) return;  // add(x, zero) == x
        const int j = (c >> 5) - wb;
        const int rk = (int)pre16[j] + __popc(bm[j] & ((1u << (c & 31)) - 1u));
        atomic_accumulate<SR, true>(&acc[rk], v);
      });
      __syncthreads();
    }
    // 4. values out (zero() entries counted for the drop-zeros fix-up)
    int zc = 0;
    for (int e = threadIdx.x; e < nr; e += THREADS) zc += SR::is_zero(acc[e]) ? 1 : 0;
    smem_values_out<V>(cvals, base + r0, acc, nr, threadIdx.x, THREADS);
    const int zt = Red(tmp.red).Sum(zc);
    if (threadIdx.x == 0 && zt > 0) {
      atomicAdd(rowzero + i, (unsigned long long)zt);
      atomicAdd(zeros, (unsigned long long)zt);
    }
    __syncthreads();
  }
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
