// Row-accumulation kernels shared by the local multiply (esc_multiply
// replacement, local_spgemm.hpp:83-156) and the partial merge
// (merge_partials replacement, summa.hpp:122-172).
//
// Both operations have the same shape: output row i is the semiring fold of
// a list of SEGMENTS, each a column-sorted run of (column, value) items from
// some CSR row, optionally multiplied on the left by a scalar:
//   local multiply:  segments of row i = rows k of R for each L entry (i, k),
//                    item = mul(l_ik, r_kj)                     (Gustavson)
//   merge:           segments of row i = row i of each partial, item = value
// (the merge is the product [I I .. I] * vstack(partials)).  A Source type
// describes the segments; the kernels below are written once against it.
//
// Items are enumerated warp-cooperatively and FLATTENED across segments: a
// warp takes 32 segments, scans their lengths with shuffles, and each lane
// locates its item by a 5-step shuffle binary search, so R-MAT's short rows
// (median ~4 entries) still keep all 32 lanes busy.  In the CTA-per-row
// kernels the row's products are first split into equal per-warp shares
// (merge-path over a shared-memory prefix of the segment lengths).
//
// Pipeline (one call):
//   K1 analyse : per-row product count F_i, bound U_i = min(F_i, ncols), bin
//   K2 bin     : scatter rows into per-bin lists (dense bin sorted by F desc)
//   K4 numeric, per bin, on concurrent streams:
//      bin 1   F <= 32        warp-ESC: products in registers, 32-lane bitonic
//                             sort on (col, product#), segmented shuffle fold
//      bin 2   F <= 512       block-ESC: products placed in product order in
//                             shared memory, stable block radix sort on the
//                             column, segmented block scan folds each run
//                             (deterministic fold order)
//      bin 3,4 U <= 4096      shared-memory hash (4K / 8K slots), atomic fold,
//                             bitonic sort of the occupied slots
//      bin 6   long rows      dense accumulator over column PANELS of width W
//                             in shared memory (128 KB), native smem atomics,
//                             presence = value != zero() scanned in order ->
//                             sorted output, accumulator restored while
//                             scanning (no clears); per-row segment
//                             descriptors cached in smem across panels
//      bin 7   long rows of   largest shared-memory hash, when panels would
//              very wide C    be mostly empty
//      every row writes a scratch slot of U_i entries and reports nnz_i
//   K7 compact : rowptr = scan(nnz); copy scratch -> exact-size CSR
//   (when the scratch would not fit: a counting pass, exact rowptr, and a
//    second pass writing straight into C)
#pragma once
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "semiring.cuh"

namespace spg {

constexpr int kNumBins = 12;
constexpr int32_t kEmptyKey = -1;
constexpr unsigned kFull = 0xffffffffu;

enum Bin : uint8_t {
  kBinEmpty = 0,
  kBinWarpEsc = 1,   // F <= 32
  kBinEsc512 = 2,    // F <= 512: block-ESC
  kBinHash4K = 3,    // U <= 2048: 4K-slot hash
  kBinHash8K = 4,    // U <= 4096: 8K-slot hash
  kBinHash2K = 5,    // U <= 1024: 2K-slot hash, 128 threads (many CTAs per SM)
  kBinDense = 6,     // long rows: dense column panels
  kBinHashMax = 7,   // wide outputs: largest smem hash
  kBinBitRank = 8,   // F <= kBitRankMax, narrow C: presence bitmap + ranked accumulator
  kBinRankPanels = 9,  // longer rows in a bounded column window: bitmap ranks, accumulator panels in rank space
  kBinBitmap = 10,     // bitmap-rank pipeline (bitmap_rank.cuh): symbolic bitmap pass, then ranks, output direct into C
  kBinWide = 11,       // dense-bin rows whose panels do not fit (very wide outputs): sort fallback (wide_rows.cuh)
};

// ---------------------------------------------------------------------------
// Sources
// ---------------------------------------------------------------------------
template <class SR>
struct MulSource {
  using V = typename SR::value_type;
  static constexpr bool kMultiSrc = false;
  const int64_t* lptr;
  const int32_t* lidx;
  const V* lval;
  const int64_t* rptr;
  const int32_t* ridx;
  const V* rval;
  int64_t nrows;
  // panel offsets: poff[k * (npanels + 1) + p] = first entry of R row k with
  // column >= p * W, relative to rptr[k] (only when npanels > 1)
  const int32_t* poff = nullptr;
  int npanels = 1;

  __device__ __forceinline__ int64_t seg_begin(int64_t i) const { return lptr[i]; }
  __device__ __forceinline__ int64_t seg_end(int64_t i) const { return lptr[i + 1]; }
  __device__ __forceinline__ int64_t seg_len(int64_t, int64_t s) const {
    const int32_t k = __ldg(lidx + s);
    return __ldg(rptr + k + 1) - __ldg(rptr + k);
  }
  // segment s of row i restricted to panel p (p < 0: whole segment)
  __device__ __forceinline__ void seg(int64_t, int64_t s, int p, int64_t& b, int& len, int& sid, V& mult) const {
    const int32_t k = __ldg(lidx + s);
    b = __ldg(rptr + k);
    if (p < 0) {
      len = (int)(__ldg(rptr + k + 1) - b);
    } else {
      const int32_t* po = poff + (int64_t)k * (npanels + 1) + p;
      const int32_t lo = __ldg(po), hi = __ldg(po + 1);
      b += lo;
      len = hi - lo;
    }
    sid = 0;
    mult = lval[s];
  }
  // panel offsets of segment s (relative to its start b) into out[0 .. np]
  __device__ __forceinline__ void panel_offsets(int64_t, int64_t s, int64_t, int, int32_t* out, int np) const {
    const int32_t k = __ldg(lidx + s);
    const int32_t* po = poff + (int64_t)k * (np + 1);
    for (int q = 0; q <= np; ++q) out[q] = __ldg(po + q);
  }
  __device__ __forceinline__ int32_t col(int, int64_t u) const { return __ldg(ridx + u); }
  __device__ __forceinline__ V val(int, int64_t u) const { return rval[u]; }
  __device__ __forceinline__ V item(const V& mult, const V& v) const { return SR::mul(mult, v); }
};

constexpr int kMaxMergeParts = 64;
struct MergeParts {
  const int64_t* ptr[kMaxMergeParts];
  const int32_t* idx[kMaxMergeParts];
  const void* val[kMaxMergeParts];
};

template <class SR>
struct MergeSource {
  using V = typename SR::value_type;
  static constexpr bool kMultiSrc = true;
  MergeParts p;
  int nparts;
  int64_t nrows;
  int panel_w = 0;  // panel width for the dense bin (found by binary search)

  __device__ __forceinline__ int64_t seg_begin(int64_t) const { return 0; }
  __device__ __forceinline__ int64_t seg_end(int64_t) const { return nparts; }
  __device__ __forceinline__ int64_t seg_len(int64_t i, int64_t s) const {
    const int64_t* ptr = p.ptr[s];
    return ptr[i + 1] - ptr[i];
  }
  __device__ __forceinline__ static int64_t lower_bound(const int32_t* a, int64_t lo, int64_t hi, int64_t x) {
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)a[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    return lo;
  }
  __device__ __forceinline__ void seg(int64_t i, int64_t s, int pnl, int64_t& b, int& len, int& sid, V& mult) const {
    const int64_t* ptr = p.ptr[s];
    int64_t lo = ptr[i], hi = ptr[i + 1];
    if (pnl >= 0) {
      const int32_t* ix = p.idx[s];
      const int64_t f = lower_bound(ix, lo, hi, (int64_t)pnl * panel_w);
      hi = lower_bound(ix, f, hi, (int64_t)(pnl + 1) * panel_w);
      lo = f;
    }
    b = lo;
    len = (int)(hi - lo);
    sid = (int)s;
    mult = SR::one();
  }
  __device__ __forceinline__ void panel_offsets(int64_t, int64_t s, int64_t b, int len, int32_t* out, int np) const {
    const int32_t* ix = p.idx[s];
    int64_t lo = b;
    for (int q = 0; q <= np; ++q) {
      lo = lower_bound(ix, lo, b + len, (int64_t)q * panel_w);
      out[q] = (int32_t)(lo - b);
    }
  }
  __device__ __forceinline__ int32_t col(int sid, int64_t u) const { return p.idx[sid][u]; }
  __device__ __forceinline__ V val(int sid, int64_t u) const { return static_cast<const V*>(p.val[sid])[u]; }
  __device__ __forceinline__ V item(const V&, const V& v) const { return v; }
};

// ---------------------------------------------------------------------------
// Geometry per value width
// ---------------------------------------------------------------------------
template <class V>
struct Geom {
  // hash tables: largest table whose keys + values fit in ~200 KB of smem
  static constexpr int kMaxT = sizeof(V) <= 4 ? 16384 : 8192;
  // dense panel width: 128 KB of accumulator values (64K columns for bool)
  static constexpr int kPanelW = (131072 / (int)sizeof(V)) > 65536 ? 65536 : (131072 / (int)sizeof(V));
};
constexpr int kDenseMaxPanels = 16;   // beyond this many panels prefer hashing
constexpr int kDenseMinPerPanel = 1024;
constexpr int64_t kDenseMinRow = 4096;  // rows with more products go dense (when panels are few)
#ifndef SPG_BITRANK_MINF
#define SPG_BITRANK_MINF 2048
#endif
constexpr int64_t kBitRankMinF = SPG_BITRANK_MINF;  // bit-rank bin floor (smaller rows: hash bins, more rows per SM)

template <class V>
__host__ __device__ inline int npanels_for(int64_t ncols, int w = Geom<V>::kPanelW) {
  return (int)((ncols + w - 1) / w);
}

// ---------------------------------------------------------------------------
// Value shuffles (any width)
// ---------------------------------------------------------------------------
template <class V>
__device__ __forceinline__ V shfl_v(const V& v, int src) {
  if constexpr (sizeof(V) < 4) {
    const uint32_t w = __shfl_sync(kFull, (uint32_t)(*reinterpret_cast<const uint8_t*>(&v)), src);
    V out;
    *reinterpret_cast<uint8_t*>(&out) = (uint8_t)w;
    return out;
  } else {
    constexpr int W = sizeof(V) / 4;
    uint32_t w[W];
    memcpy(w, &v, sizeof(V));
#pragma unroll
    for (int k = 0; k < W; ++k) w[k] = __shfl_sync(kFull, w[k], src);
    V out;
    memcpy(&out, w, sizeof(V));
    return out;
  }
}
template <class V>
__device__ __forceinline__ V shfl_xor_v(const V& v, int m) {
  return shfl_v(v, (threadIdx.x & 31) ^ m);
}
template <class V>
__device__ __forceinline__ V shfl_up_v(const V& v, int d) {
  const int lane = threadIdx.x & 31;
  return shfl_v(v, lane >= d ? lane - d : lane);
}

// ---------------------------------------------------------------------------
// Flattened warp enumeration of the items of segments [s0, s1) of row i
// (panel p, or whole segments for p < 0), warps striding by `sstride`
// segments.  f(col, value, seg_index, offset_in_segment) is called once per
// item; every lane of the warp must call this.
// ---------------------------------------------------------------------------
template <class SR, class Src, class F>
__device__ __forceinline__ void warp_items(const Src& src, int64_t i, int64_t s0, int64_t s1, int p, int64_t sstride,
                                           F&& f) {
  using V = typename SR::value_type;
  const int lane = threadIdx.x & 31;
  for (int64_t base = s0; base < s1; base += sstride) {
    const int64_t s = base + lane;
    int64_t b = 0;
    int len = 0, sid = 0;
    V mult = SR::zero();
    if (s < s1) src.seg(i, s, p, b, len, sid, mult);
    int incl = len;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += t;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    const int excl = incl - len;
    for (int q0 = 0; q0 < total; q0 += 32) {
      const int q = q0 + lane;
      int pos = 0;
#pragma unroll
      for (int step = 16; step >= 1; step >>= 1) {
        const int v = __shfl_sync(kFull, incl, pos + step - 1);
        if (v <= q) pos += step;
      }
      const long long bb = __shfl_sync(kFull, (long long)b, pos);
      const int ex = __shfl_sync(kFull, excl, pos);
      const V m = shfl_v(mult, pos);
      int sd = 0;
      if constexpr (Src::kMultiSrc) sd = __shfl_sync(kFull, sid, pos);
      if (q < total) {
        const int off = q - ex;
        const int64_t u = bb + off;
        f(src.col(sd, u), src.item(m, src.val(sd, u)), base + pos, off);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K1: per-row analysis and binning policy
// ---------------------------------------------------------------------------
template <class SR, class Src>
__global__ void __launch_bounds__(256) analyse_rows_kernel(Src src, int64_t ncols_out, int64_t dense_min,
                                                           int64_t bitrank_max, int64_t bitrank_segs,
                                                           int64_t bitrank_span, int64_t rankpanel_segs,
                                                           int64_t rankpanel_maxf, int64_t bitmap_min,
                                                           int32_t* __restrict__ colmin,
                                                           int64_t* __restrict__ prods,
                                                           int64_t* __restrict__ ubound,
                                                           uint8_t* __restrict__ bins) {
  using V = typename SR::value_type;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int np = npanels_for<V>(ncols_out);
  for (int64_t i = warp; i < src.nrows; i += nwarps) {
    const int64_t sb = src.seg_begin(i), se = src.seg_end(i);
    int64_t f = 0;
    for (int64_t s = sb + lane; s < se; s += 32) f += src.seg_len(i, s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) f += __shfl_xor_sync(kFull, f, o);
    // column window of the row (bit-rank candidates only): min first / max last column over its segments
    int64_t span = INT64_MAX;
    if (bitrank_max > 0 && f > kBitRankMinF &&
        ((f <= bitrank_max && se - sb <= bitrank_segs) ||
         (rankpanel_segs > 0 && f <= rankpanel_maxf && se - sb <= rankpanel_segs))) {
      int32_t cmin = INT32_MAX, cmax = -1;
      for (int64_t s = sb + lane; s < se; s += 32) {
        int64_t bb;
        int len, sd;
        V m;
        src.seg(i, s, -1, bb, len, sd, m);
        if (len > 0) {
          cmin = min(cmin, src.col(sd, bb));
          cmax = max(cmax, src.col(sd, bb + len - 1));
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        cmin = min(cmin, __shfl_xor_sync(kFull, cmin, o));
        cmax = max(cmax, __shfl_xor_sync(kFull, cmax, o));
      }
      span = cmax >= cmin ? (int64_t)cmax - cmin + 1 : 0;
      if (lane == 0) colmin[i] = cmin;
    }
    if (lane == 0) {
      const int64_t u = f < ncols_out ? f : ncols_out;
      const int64_t nseg = se - sb;
      uint8_t b;
      const bool dense_ok = np <= kDenseMaxPanels || f >= (int64_t)kDenseMinPerPanel * np;
      if (f == 0) b = kBinEmpty;
      else if (bitmap_min > 0 && f > bitmap_min) b = kBinBitmap;
      else if (f <= 32) b = kBinWarpEsc;
      else if (f <= 512 && nseg <= 512) b = kBinEsc512;
      else if (bitrank_max > 0 && f <= bitrank_max && nseg <= bitrank_segs && span <= bitrank_span) b = kBinBitRank;
      else if (rankpanel_segs > 0 && f > bitrank_max && f <= rankpanel_maxf && nseg <= rankpanel_segs &&
               span <= bitrank_span)
        b = kBinRankPanels;
      else if (f > dense_min && dense_ok) b = kBinDense;
      else if (u <= 1024) b = kBinHash2K;
      else if (u <= 2048) b = kBinHash4K;
      else if (u <= 4096) b = kBinHash8K;
      else if (u <= Geom<V>::kMaxT / 2) b = kBinHashMax;
      else b = kBinDense;
      prods[i] = f;
      ubound[i] = (b == kBinEmpty || b == kBinBitmap) ? 0 : ((u + 3) & ~int64_t(3));  // 16-byte aligned scratch slots
      bins[i] = b;
    }
  }
}

// number of rows (prefix of a list sorted by F descending) with more than t products
static __global__ void count_above_kernel(const int64_t* __restrict__ rows, int64_t n, const int64_t* __restrict__ f,
                                          int64_t t, unsigned long long* out) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    if (f[rows[k]] > t) atomicAdd(out, 1ull);
}

// ---------------------------------------------------------------------------
// K2: bin histogram + scatter into per-bin row lists
// ---------------------------------------------------------------------------
static __global__ void __launch_bounds__(1024) bin_count_kernel(const uint8_t* __restrict__ bins, int64_t n,
                                                                 unsigned long long* counts) {
  __shared__ unsigned int h[kNumBins];
  if (threadIdx.x < kNumBins) h[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[bins[i]], 1u);
  __syncthreads();
  if (threadIdx.x < kNumBins && h[threadIdx.x])
    atomicAdd(&counts[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}

static __global__ void __launch_bounds__(1024) bin_scatter_kernel(const uint8_t* __restrict__ bins, int64_t n,
                                                                   unsigned long long* cursor,
                                                                   int64_t* __restrict__ lists) {
  __shared__ unsigned int h[kNumBins];
  __shared__ unsigned long long base[kNumBins];
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x < kNumBins) h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t i = c + threadIdx.x;
    int b = -1;
    unsigned int slot = 0;
    if (i < n) {
      b = bins[i];
      if (b != kBinEmpty) slot = atomicAdd(&h[b], 1u);
    }
    __syncthreads();
    if (threadIdx.x < kNumBins)
      base[threadIdx.x] = h[threadIdx.x] ? atomicAdd(&cursor[threadIdx.x], (unsigned long long)h[threadIdx.x]) : 0;
    __syncthreads();
    if (b > 0) lists[base[b] + slot] = i;
    __syncthreads();
  }
}

static __global__ void zero_empty_rows_kernel(const uint8_t* __restrict__ bins, int64_t n, int64_t* __restrict__ rownnz) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (bins[i] == kBinEmpty) rownnz[i] = 0;
}

// keys[k] = prods[rows[k]] (to sort the dense bin by work, largest first)
static __global__ void gather_keys_kernel(const int64_t* __restrict__ rows, int64_t n, const int64_t* __restrict__ prods,
                                          int64_t* __restrict__ keys) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
    keys[k] = prods[rows[k]];
}

// Panel offsets of every R row: poff[k*(np+1) + p] = #entries of row k with
// column < p * W  (warp per row, lanes binary-search the boundaries).
static __global__ void __launch_bounds__(256) panel_offsets_kernel(int64_t nrows, const int64_t* __restrict__ rptr,
                                                                   const int32_t* __restrict__ ridx, int np, int W,
                                                                   int32_t* __restrict__ poff) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t k = warp; k < nrows; k += nwarps) {
    const int64_t b = rptr[k], e = rptr[k + 1];
    for (int p = lane; p <= np; p += 32) {
      const int64_t x = (int64_t)p * W;
      int64_t lo = b, hi = e;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if ((int64_t)ridx[mid] < x) lo = mid + 1;
        else hi = mid;
      }
      poff[k * (np + 1) + p] = (int32_t)(lo - b);
    }
  }
}

// ---------------------------------------------------------------------------
// Where the row kernels put their output.
//  * direct: row i starts at off[i] (the exact rowptr of C in the second
//    pass of two-pass mode);
//  * exact claim ("bump"): a row, once its nnz is known, claims exactly that
//    many entries of the scratch with one atomicAdd; dense rows claim one
//    chunk per column panel.  Scratch holds nnz(C) entries, not the
//    products bound; a claim past `cap` is not stored (overflow => the
//    driver reruns in direct mode with the exact rowptr it now has);
//  * cols == nullptr: count only.
// ---------------------------------------------------------------------------
template <class V>
struct RowOut {
  int32_t* cols = nullptr;
  V* vals = nullptr;
  const int64_t* off = nullptr;
  unsigned long long* bump = nullptr;
  int64_t cap = 0;
  int64_t* rowstart = nullptr;  // claim mode: scratch start of row i (-2: dense row, see chunks)
  int64_t* chunks = nullptr;    // claim mode, dense rows: (start, count) per (dense slot, panel)
  int64_t slot_base = 0;        // dense slot of the launch's first row (several dense launches share `chunks`)
  int chunk_stride = 0;         // chunk entries per dense slot (>= the launch's panel count)
  // U-slot mode, dense rows: per-(panel, warp) chunks inside the row's slot
  // ((start within the slot, count) per chunk; a row's chunks in (panel,
  // warp) order are its sorted output) — warps claim without a block scan
  int32_t* wchunks = nullptr;
  int wstride = 0;              // chunks per dense slot = panels x warps
  int64_t* rownnz = nullptr;

  __device__ __forceinline__ bool writes() const { return cols != nullptr; }
  __device__ __forceinline__ int64_t claim(int64_t n) const {
    const unsigned long long b = n ? atomicAdd(bump, (unsigned long long)n) : 0ull;
    return (int64_t)b + n <= cap ? (int64_t)b : -1;
  }
  // base of row i's n entries; -1 = do not store
  __device__ __forceinline__ int64_t claim_row(int64_t i, int64_t n) const {
    if (!cols) return -1;
    if (!bump) return off[i];
    const int64_t b = claim(n);
    rowstart[i] = b;
    return b;
  }
  // base of dense row i's panel p chunk (n entries, `written` before it)
  __device__ __forceinline__ int64_t claim_chunk(int64_t i, int64_t slot, int p, int np, int64_t written,
                                                 int64_t n) const {
    if (!cols) return -1;
    if (!bump) return off[i] + written;
    const int64_t b = claim(n);
    const int64_t e = (slot + slot_base) * (chunk_stride > 0 ? chunk_stride : np) + p;
    chunks[2 * e] = b;
    chunks[2 * e + 1] = n;
    return b;
  }
};

// ---------------------------------------------------------------------------
// K4 bin 1: warp-ESC for rows with <= 32 products
// ---------------------------------------------------------------------------
template <class SR, class Src>
__global__ void __launch_bounds__(256) esc_warp_kernel(Src src, const int64_t* __restrict__ rows, int64_t nrows_bin,
                                                       RowOut<typename SR::value_type> out) {
  using V = typename SR::value_type;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < nrows_bin; r += nwarps) {
    const int64_t i = rows[r];
    uint64_t key = ~0ull;  // (col << 32) | product#  ; ~0 = no item
    V val = SR::zero();
    // every product lands on its own lane, in product order (<= 32 of them)
    warp_items<SR>(src, i, src.seg_begin(i), src.seg_end(i), -1, 32,
                   [&](int32_t c, const V& v, int64_t, int) {
                     key = ((uint64_t)(uint32_t)c << 32) | (uint32_t)lane;
                     val = v;
                   });
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        const uint64_t okey = __shfl_xor_sync(kFull, key, j);
        const V oval = shfl_xor_v(val, j);
        const bool up = (lane & k) == 0;
        const bool lower = (lane & j) == 0;
        const bool take = (lower == up) ? (okey < key) : (okey > key);
        if (take) {
          key = okey;
          val = oval;
        }
      }
    }
    const uint32_t col = (uint32_t)(key >> 32);
    const bool valid = key != ~0ull;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t ocol = __shfl_up_sync(kFull, col, d);
      const V oval = shfl_up_v(val, d);
      if (lane >= d && ocol == col) val = SR::add(oval, val);
    }
    const uint32_t ncol = __shfl_down_sync(kFull, col, 1);
    const bool tail = valid && (lane == 31 || ncol != col);
    const bool keep = tail && !SR::is_zero(val);
    const unsigned m = __ballot_sync(kFull, keep);
    const int pos = __popc(m & ((1u << lane) - 1));
    int64_t o = 0;
    if (lane == 0) {
      o = out.claim_row(i, __popc(m));
      out.rownnz[i] = __popc(m);
    }
    o = __shfl_sync(kFull, o, 0);
    if (keep && o >= 0) {
      out.cols[o + pos] = (int32_t)col;
      out.vals[o + pos] = val;
    }
  }
}

// ---------------------------------------------------------------------------
// K4 bins 2-4: block-ESC.  Products of one row are placed in product order
// (segment-major) in shared memory, stably radix-sorted by column, and each
// run of equal columns is folded by a segmented block scan.
// ---------------------------------------------------------------------------
template <class SR>
struct SegFold {
  using V = typename SR::value_type;
  struct T {
    V v;
    int head;
  };
  __device__ __forceinline__ T operator()(const T& a, const T& b) const {
    T r;
    r.head = a.head | b.head;
    r.v = b.head ? b.v : SR::add(a.v, b.v);
    return r;
  }
};

template <class SR, int THREADS, int ITEMS>
struct EscSmem {
  using V = typename SR::value_type;
  static constexpr int CAP = THREADS * ITEMS;
  using Sort = cub::BlockRadixSort<uint32_t, THREADS, ITEMS, uint16_t, 6>;
  using Fold = cub::BlockScan<typename SegFold<SR>::T, THREADS>;
  using Count = cub::BlockScan<int, THREADS>;
  union {
    typename Sort::TempStorage sort;
    typename Fold::TempStorage fold;
    typename Count::TempStorage count;
  } tmp;
  uint32_t keys[CAP];
  V vals[CAP];
  int seg_off[CAP + 1];  // exclusive prefix of segment lengths (<= CAP segments)
  uint32_t run_cols[CAP + 1];
};

template <class SR, class Src, int THREADS, int ITEMS>
__global__ void __launch_bounds__(THREADS) esc_block_kernel(Src src, const int64_t* __restrict__ rows,
                                                            int64_t nrows_bin, int end_bit,
                                                            RowOut<typename SR::value_type> out) {
  using V = typename SR::value_type;
  using S = EscSmem<SR, THREADS, ITEMS>;
  __shared__ long long s_base;
  constexpr int NW = THREADS / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S& sm = *reinterpret_cast<S*>(smem_raw);
  const int wid = threadIdx.x >> 5;

  for (int64_t r = blockIdx.x; r < nrows_bin; r += gridDim.x) {
    const int64_t i = rows[r];
    const int64_t sb = src.seg_begin(i), se = src.seg_end(i);
    const int nseg = (int)(se - sb);  // <= CAP for these bins
    // 1. exclusive prefix of segment lengths (product order = segment order)
    int lens[ITEMS];
    int local = 0;
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      const int s = threadIdx.x * ITEMS + q;
      lens[q] = s < nseg ? (int)src.seg_len(i, sb + s) : 0;
      local += lens[q];
    }
    int first, total;
    typename S::Count(sm.tmp.count).ExclusiveSum(local, first, total);
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      const int s = threadIdx.x * ITEMS + q;
      if (s < nseg) sm.seg_off[s] = first;
      first += lens[q];
    }
    __syncthreads();
    // 2. expand: each product lands at seg_off[s] + offset-in-segment
    warp_items<SR>(src, i, sb + wid * 32, se, -1, (int64_t)NW * 32,
                   [&](int32_t c, const V& v, int64_t s, int o) {
                     const int pos = sm.seg_off[s - sb] + o;
                     sm.keys[pos] = (uint32_t)c;
                     sm.vals[pos] = v;
                   });
    __syncthreads();
    // 3. stable radix sort of (column -> product index), blocked arrangement
    uint32_t k[ITEMS];
    uint16_t idx[ITEMS];
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      const int e = threadIdx.x * ITEMS + q;
      k[q] = e < total ? sm.keys[e] : (1u << end_bit);  // padding sorts last
      idx[q] = (uint16_t)e;
    }
    __syncthreads();
    typename S::Sort(sm.tmp.sort).Sort(k, idx, 0, end_bit + 1);
    __syncthreads();
    // 4. segmented fold of equal-column runs
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) sm.run_cols[threadIdx.x * ITEMS + q] = k[q];
    if (threadIdx.x == 0) sm.run_cols[S::CAP] = 0xffffffffu;
    __syncthreads();
    typename SegFold<SR>::T t[ITEMS];
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      const int e = threadIdx.x * ITEMS + q;
      t[q].head = (e == 0 || sm.run_cols[e - 1] != k[q]) ? 1 : 0;
      t[q].v = e < total ? sm.vals[idx[q]] : SR::zero();
    }
    __syncthreads();
    typename S::Fold(sm.tmp.fold).InclusiveScan(t, t, SegFold<SR>());
    __syncthreads();
    // 5. keep run tails with non-zero value; compact in column order
    int keep[ITEMS];
    int nkeep = 0;
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      const int e = threadIdx.x * ITEMS + q;
      const bool tail = e < total && sm.run_cols[e + 1] != k[q];
      keep[q] = (tail && !SR::is_zero(t[q].v)) ? 1 : 0;
      nkeep += keep[q];
    }
    int kfirst, ktotal;
    typename S::Count(sm.tmp.count).ExclusiveSum(nkeep, kfirst, ktotal);
    if (threadIdx.x == 0) {
      s_base = out.claim_row(i, ktotal);
      out.rownnz[i] = ktotal;
    }
    __syncthreads();
    const int64_t o = s_base;
#pragma unroll
    for (int q = 0; q < ITEMS; ++q) {
      if (keep[q]) {
        if (o >= 0) {
          out.cols[o + kfirst] = (int32_t)k[q];
          out.vals[o + kfirst] = t[q].v;
        }
        ++kfirst;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Per-row staging of segment descriptors in shared memory + balanced
// (merge-path) enumeration: the row's products are split into NW equal
// shares, one per warp, so a row with few segments still occupies every
// warp of the CTA (warp-per-32-segments left most warps idle at the barrier).
// ---------------------------------------------------------------------------
template <class SR, class Src>
struct SegCache {
  using V = typename SR::value_type;
  int64_t* b;    // [cap] start of the segment (whole row)
  int32_t* sid;  // [cap] source id (multi-source merges)
  V* mult;       // [cap]
  int32_t* po;   // [cap * (np + 1)] panel offsets relative to b (np > 1), or [cap] lengths (np == 1)
  int32_t* pre;  // [cap + 1] exclusive prefix of the (panel) lengths
  int np;

  static __host__ __device__ size_t bytes_per_seg(int npanels) {
    return sizeof(int64_t) + sizeof(int32_t) + sizeof(V) + sizeof(int32_t) * (npanels == 1 ? 1 : npanels + 1) +
           sizeof(int32_t);
  }
  // carve the cache out of `base` for `cap` segments
  __device__ __forceinline__ void carve(unsigned char* base, int cap, int npanels) {
    np = npanels;
    b = reinterpret_cast<int64_t*>(base);
    sid = reinterpret_cast<int32_t*>(b + cap);
    mult = reinterpret_cast<V*>(reinterpret_cast<unsigned char*>(sid) + ((sizeof(int32_t) * cap + 15) & ~size_t(15)));
    po = reinterpret_cast<int32_t*>(reinterpret_cast<unsigned char*>(mult) + ((sizeof(V) * cap + 15) & ~size_t(15)));
    pre = po + (size_t)cap * (np == 1 ? 1 : np + 1);
  }
  __device__ __forceinline__ void load(const Src& src, int64_t i, int64_t s0, int n, int tid, int nthreads) const {
    for (int t = tid; t < n; t += nthreads) {
      int64_t bb;
      int len, sd;
      V m;
      src.seg(i, s0 + t, -1, bb, len, sd, m);
      b[t] = bb;
      sid[t] = sd;
      mult[t] = m;
      if (np == 1) po[t] = len;
      else src.panel_offsets(i, s0 + t, bb, len, po + (int64_t)t * (np + 1), np);
    }
  }
  __device__ __forceinline__ int len(int t, int p) const {
    if (np == 1) return po[t];
    const int32_t* q = po + (int64_t)t * (np + 1) + p;
    return q[1] - q[0];
  }
  __device__ __forceinline__ void get(int t, int p, int64_t& bb, int& ln, int& sd, V& m) const {
    m = mult[t];
    sd = sid[t];
    if (np == 1) {
      bb = b[t];
      ln = po[t];
    } else {
      const int32_t* q = po + (int64_t)t * (np + 1) + p;
      bb = b[t] + q[0];
      ln = q[1] - q[0];
    }
  }
  // pre[0..n] = exclusive prefix of len(t, p); returns the total.  Block-wide.
  template <int THREADS, class Scan>
  __device__ __forceinline__ int prefix(int n, int p, typename Scan::TempStorage& tmp) const {
    const int ipt = (n + THREADS - 1) / THREADS;
    const int t0 = threadIdx.x * ipt;
    int local = 0;
    for (int q = 0; q < ipt; ++q) {
      const int t = t0 + q;
      if (t < n) local += len(t, p);
    }
    int first, total;
    Scan(tmp).ExclusiveSum(local, first, total);
    for (int q = 0; q < ipt; ++q) {
      const int t = t0 + q;
      if (t < n) {
        pre[t] = first;
        first += len(t, p);
      }
    }
    if (threadIdx.x == 0) pre[n] = total;
    __syncthreads();
    return total;
  }
};

// Position of the k-th (0-based) set bit of x (k < popc(x)); popc bisection.
__device__ __forceinline__ int nth_set_bit(uint32_t x, int k) {
  int pos = 0;
  int c = __popc(x & 0xffffu);
  if (k >= c) { k -= c; pos += 16; x >>= 16; }
  c = __popc(x & 0xffu);
  if (k >= c) { k -= c; pos += 8; x >>= 8; }
  c = __popc(x & 0xfu);
  if (k >= c) { k -= c; pos += 4; x >>= 4; }
  c = __popc(x & 0x3u);
  if (k >= c) { k -= c; pos += 2; x >>= 2; }
  c = (int)(x & 1u);
  if (k >= c) pos += 1;
  return pos;
}

// Warp `wid` of NW enumerates its equal share of the cached segments' items
// (panel p); f(col, value) per item, two items per lane in flight.
// kNarrowSearch: bound each batch's shuffle search to the segments [f, l]
// it touches (measured: a gain for the long segments of dense rows, a loss
// for short ones — used by the dense kernel only).
template <class SR, class Src, int NW, int IPL = 2, bool kColsOnly = false, bool kNarrowSearch = false, class F>
__device__ __forceinline__ void balanced_items(const Src& src, const SegCache<SR, Src>& c, int n, int p, F&& f) {
  using V = typename SR::value_type;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int P = c.pre[n];
  const int lo_q = (int)((int64_t)P * wid / NW), hi_q = (int)((int64_t)P * (wid + 1) / NW);
  if (lo_q >= hi_q) return;
  int s = 0, hs = n;  // largest s with pre[s] <= lo_q
  while (hs - s > 1) {
    const int mid = (s + hs) >> 1;
    if (c.pre[mid] <= lo_q) s = mid;
    else hs = mid;
  }
  for (int s0 = s; s0 < n && c.pre[s0] < hi_q; s0 += 32) {
    const int t = s0 + lane;
    int64_t bb = 0;
    int L = 0, sd = 0;
    V m = SR::zero();
    if (t < n) {
      int ln;
      c.get(t, p, bb, ln, sd, m);
      const int st = c.pre[t];
      const int beg = st > lo_q ? st : lo_q;
      const int end = (st + ln) < hi_q ? (st + ln) : hi_q;
      L = end > beg ? end - beg : 0;
      bb += beg - st;
    }
    int incl = L;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int x = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += x;
    }
    const int total = __shfl_sync(kFull, incl, 31);
    const int excl = incl - L;
    for (int q0 = 0; q0 < total; q0 += 32 * IPL) {
      int pos[IPL];
      if constexpr (kNarrowSearch) {
        // the batch's items lie in segments [f, l]: search only that range
        // (one segment: no shuffle at all; two: one step)
        const int qlast = min(q0 + 32 * IPL - 1, total - 1);
        const int f = __popc(__ballot_sync(kFull, incl <= q0));
        const int l = __popc(__ballot_sync(kFull, incl <= qlast));
#pragma unroll
        for (int u = 0; u < IPL; ++u) pos[u] = f;
        const int span = l - f;
        if (span > 0) {
          for (int step = 1 << (31 - __clz(span)); step >= 1; step >>= 1) {
#pragma unroll
            for (int u = 0; u < IPL; ++u) {
              const int at = pos[u] + step - 1;
              const int v = __shfl_sync(kFull, incl, at < 31 ? at : 31);
              if (at < l && v <= q0 + 32 * u + lane) pos[u] += step;
            }
          }
        }
      } else {
#pragma unroll
        for (int u = 0; u < IPL; ++u) pos[u] = 0;
#pragma unroll
        for (int step = 16; step >= 1; step >>= 1) {
#pragma unroll
          for (int u = 0; u < IPL; ++u) {
            const int v = __shfl_sync(kFull, incl, pos[u] + step - 1);
            if (v <= q0 + 32 * u + lane) pos[u] += step;
          }
        }
      }
      int32_t cc[IPL];
      V xx[IPL], mm[IPL];
#pragma unroll
      for (int u = 0; u < IPL; ++u) {
        const int q = q0 + 32 * u + lane;
        const long long bu = __shfl_sync(kFull, (long long)bb, pos[u]);
        const int eu = __shfl_sync(kFull, excl, pos[u]);
        mm[u] = shfl_v(m, pos[u]);
        int su = 0;
        if constexpr (Src::kMultiSrc) su = __shfl_sync(kFull, sd, pos[u]);
        if (q < total) {
          const int64_t w = bu + (q - eu);
          cc[u] = src.col(su, w);
          if constexpr (!kColsOnly) xx[u] = src.val(su, w);
        }
      }
#pragma unroll
      for (int u = 0; u < IPL; ++u)
        if (q0 + 32 * u + lane < total) {
          if constexpr (kColsOnly) f(cc[u], mm[u]);  // value not loaded
          else f(cc[u], src.item(mm[u], xx[u]));
        }
    }
  }
}

// ---------------------------------------------------------------------------
// Ordered emission of a W-wide smem accumulator driven by its first-touch
// bitmap (one bit per column, W/32 words; warp w owns a contiguous slice of
// W/32/NW words).  Output entries are FLATTENED across lanes: a warp scans the
// popcounts of 32 words, then each lane takes one output entry per step,
// finds its word with a 5-step shuffle search and its bit with __fns, so the
// stores are coalesced and no lane idles on a sparse word.  Positions:
// block scan over the warps' counts.  Restores zero() and clears the bitmap.
// Only items != zero() ever set a bit, so the bitmap count is exact unless
// the fold can cancel back to zero() (fp64 +), which a pre-pass handles.
// Returns the number of entries written.
// ---------------------------------------------------------------------------

// Can the fold cancel back to zero() (a + (-a) == 0)?  A semiring may say so
// with `static constexpr bool add_can_cancel`; otherwise only the built-in
// arithmetic (+, x) semiring (id 0) can.
template <class SR, class = void>
struct AddCanCancelById {
  static constexpr bool value = false;
};
template <class SR>
struct AddCanCancelById<SR, decltype((void)SR::id, void())> {
  static constexpr bool value = SR::id == 0;
};
template <class SR, class = void>
struct AddCanCancel {
  static constexpr bool value = AddCanCancelById<SR>::value;
};
template <class SR>
struct AddCanCancel<SR, decltype((void)SR::add_can_cancel, void())> {
  static constexpr bool value = SR::add_can_cancel;
};

// Barrier over a warp group: BAR == 0 is __syncthreads, else named barrier
// BAR over NT threads (warp-specialised kernels).
template <int BAR, int NT>
__device__ __forceinline__ void group_sync() {
  if constexpr (BAR == 0) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"n"(BAR), "n"(NT) : "memory");
  }
}
__device__ __forceinline__ void named_sync(int bar, int nt) {
  asm volatile("bar.sync %0, %1;" ::"r"(bar), "r"(nt) : "memory");
}
__device__ __forceinline__ void named_arrive(int bar, int nt) {
  asm volatile("bar.arrive %0, %1;" ::"r"(bar), "r"(nt) : "memory");
}

template <class SR, int W, int THREADS, int BAR = 0, int WARP0 = 0>
__device__ __forceinline__ int bitmap_emit(typename SR::value_type* acc, uint32_t* bm, int col_base,
                                           const RowOut<typename SR::value_type>& out, int64_t row, int64_t slot,
                                           int panel, int npanels, int64_t written, int* wsum, long long* s_base) {
  using V = typename SR::value_type;
  constexpr int NW = THREADS / 32;
  constexpr int WORDS = W / 32;
  constexpr int WPW = WORDS / NW;  // words per warp
  constexpr int ITERS = (WPW + 31) / 32;
  static_assert(WORDS % NW == 0 && (WPW < 32 || WPW % 32 == 0), "bitmap words must split evenly over the warps");
  const int lane = threadIdx.x & 31, wid = (threadIdx.x >> 5) - WARP0;
  const int w0 = wid * WPW;
  if constexpr (AddCanCancel<SR>::value) {
    // drop touched entries whose fold cancelled to zero (restoring exact zero() bits)
    for (int it = 0; it < ITERS; ++it) {
      const int wl = it * 32 + lane;
      if (wl >= WPW) break;
      const int w = w0 + wl;
      uint32_t x = bm[w];
      for (uint32_t y = x; y; y &= y - 1) {
        const int bit = __ffs(y) - 1;
        if (SR::is_zero(acc[(w << 5) + bit])) {
          acc[(w << 5) + bit] = SR::zero();
          x &= ~(1u << bit);
        }
      }
      bm[w] = x;
    }
  }
  int cnt = 0;
  for (int it = 0; it < ITERS; ++it) {
    const int wl = it * 32 + lane;
    cnt += wl < WPW ? __popc(bm[w0 + wl]) : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
  if (lane == 0) wsum[wid] = cnt;
  group_sync<BAR, THREADS>();
  if (wid == 0) {
    const int v = lane < NW ? wsum[lane] : 0;
    int incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int t = __shfl_up_sync(kFull, incl, d);
      if (lane >= d) incl += t;
    }
    if (lane < NW) wsum[NW + lane] = incl - v;
    if (lane == 31) {
      wsum[2 * NW] = incl;
      *s_base = out.claim_chunk(row, slot, panel, npanels, written, incl);
    }
  }
  group_sync<BAR, THREADS>();
  const bool store = *s_base >= 0;
  int64_t pos = *s_base + wsum[NW + wid];
  for (int it = 0; it < ITERS; ++it) {
    const int wl = it * 32 + lane;
    const int w = w0 + wl;
    const uint32_t x = wl < WPW ? bm[w] : 0u;
    const int c = __popc(x);
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
      if (q < total) {
        const int bit = nth_set_bit(xo, q - eo);
        const int cc = ((w0 + it * 32 + own) << 5) + bit;
        if (store) {
          out.cols[pos + q] = col_base + cc;
          out.vals[pos + q] = acc[cc];
        }
        acc[cc] = SR::zero();
      }
    }
    if (x) bm[w] = 0u;
    pos += total;
  }
  const int total = wsum[2 * NW];
  group_sync<BAR, THREADS>();
  return total;
}

// Per-warp emission for U-slot mode: each warp counts the entries of its own
// column slice, claims that many slots of the row's scratch slot with one
// shared atomicAdd, records the chunk (start, count) and writes its entries
// in column order — no block-wide count/scan/offset barriers.  The chunks in
// (panel, warp) order are the row's sorted output; the compaction
// concatenates them.
template <class SR, int W, int THREADS>
__device__ __forceinline__ void bitmap_emit_warp(typename SR::value_type* acc, uint32_t* bm, int col_base,
                                                 const RowOut<typename SR::value_type>& out, int64_t row,
                                                 int64_t slot, int panel, int* s_fill) {
  using V = typename SR::value_type;
  constexpr int NW = THREADS / 32;
  constexpr int WORDS = W / 32;
  constexpr int WPW = WORDS / NW;
  constexpr int ITERS = (WPW + 31) / 32;
  static_assert(WORDS % NW == 0 && (WPW < 32 || WPW % 32 == 0), "bitmap words must split evenly over the warps");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int w0 = wid * WPW;
  if constexpr (AddCanCancel<SR>::value) {
    for (int it = 0; it < ITERS; ++it) {
      const int wl = it * 32 + lane;
      if (wl >= WPW) break;
      const int w = w0 + wl;
      uint32_t x = bm[w];
      for (uint32_t y = x; y; y &= y - 1) {
        const int bit = __ffs(y) - 1;
        if (SR::is_zero(acc[(w << 5) + bit])) {
          acc[(w << 5) + bit] = SR::zero();
          x &= ~(1u << bit);
        }
      }
      bm[w] = x;
    }
    __syncwarp();
  }
  int cnt = 0;
  for (int it = 0; it < ITERS; ++it) {
    const int wl = it * 32 + lane;
    cnt += wl < WPW ? __popc(bm[w0 + wl]) : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
  int base = 0;
  if (lane == 0) {
    base = cnt ? atomicAdd(s_fill, cnt) : 0;
    int32_t* ch = out.wchunks + 2 * ((slot + out.slot_base) * out.wstride + (int64_t)panel * NW + wid);
    ch[0] = base;
    ch[1] = cnt;
  }
  base = __shfl_sync(kFull, base, 0);
  int64_t pos = out.off[row] + base;
  for (int it = 0; it < ITERS; ++it) {
    const int wl = it * 32 + lane;
    const int w = w0 + wl;
    const uint32_t x = wl < WPW ? bm[w] : 0u;
    const int c = __popc(x);
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
      if (q < total) {
        const int bit = nth_set_bit(xo, q - eo);
        const int cc = ((w0 + it * 32 + own) << 5) + bit;
        out.cols[pos + q] = col_base + cc;
        out.vals[pos + q] = acc[cc];
        acc[cc] = SR::zero();
      }
    }
    if (x) bm[w] = 0u;
    pos += total;
  }
}

// ---------------------------------------------------------------------------
// K5 bin 6: dense accumulator over column panels in shared memory.
//
// CTAs pull rows (largest first) from a work counter.  A row's segment
// descriptors (R-row start, left scalar and the per-panel offsets) are
// gathered ONCE into shared memory; each panel re-reads them from smem while
// its products, split evenly over the warps, are folded into a W-wide
// accumulator with native smem atomics.  Presence is "value != zero()",
// exactly the reference's zero-dropping rule, so no bitmap is kept; the
// ordered scan of the accumulator emits sorted output and restores zero() as
// it goes, so no panel ever needs a separate clear.  Rows with more
// segments than the cache holds are processed in segment batches per panel.
// ---------------------------------------------------------------------------
#ifndef SPG_DENSE_IPL
#define SPG_DENSE_IPL 2
#endif
constexpr int kDenseIPL = SPG_DENSE_IPL;  // items per lane in flight in the dense product loop
#ifndef SPG_PREALL
#define SPG_PREALL 1
#endif
constexpr bool kPreAll = SPG_PREALL != 0;
template <class SR, class Src, int W, int THREADS, int MINB = 1>
__global__ void __launch_bounds__(THREADS, MINB) dense_panel_kernel(Src src, const int64_t* __restrict__ rows,
                                                              int64_t nrows_bin, int npanels, int cap,
                                                              unsigned long long* __restrict__ work,
                                                              RowOut<typename SR::value_type> out, bool preall) {
  using V = typename SR::value_type;
  constexpr int NW = THREADS / 32;
  using Count = cub::BlockScan<int, THREADS>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* acc = reinterpret_cast<V*>(smem_raw);
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem_raw + sizeof(V) * W);
  SegCache<SR, Src> cache;
  cache.carve(smem_raw + sizeof(V) * W + sizeof(uint32_t) * (W / 32), cap, npanels);
  // kPreAll: every panel's segment prefix is computed once per row (one warp
  // per panel) instead of a block scan + barrier per panel
  int* pre_all = preall ? cache.pre + ((cap + 1 + 3) & ~3) : nullptr;  // [npanels][cap + 1]
  int* const pre0 = cache.pre;
  __shared__ typename Count::TempStorage scan_tmp;
  __shared__ long long s_row, s_base;
  __shared__ int wsum[2 * NW + 1];
  __shared__ int s_fill;  // per-warp emission: entries of the current row claimed so far
  const bool warp_emit = out.wchunks != nullptr;

  for (int e = threadIdx.x; e < W; e += THREADS) acc[e] = SR::zero();
  for (int e = threadIdx.x; e < W / 32; e += THREADS) bm[e] = 0u;
  __syncthreads();
  for (;;) {
    if (threadIdx.x == 0) {
      const unsigned long long r = atomicAdd(work, 1ull);
      s_row = r < (unsigned long long)nrows_bin ? (long long)r : -1;
      s_fill = 0;
    }
    __syncthreads();
    const long long r = s_row;
    if (r < 0) break;
    const int64_t i = rows[r];
    const int64_t sb = src.seg_begin(i), se = src.seg_end(i);
    const int64_t nseg = se - sb;
    const bool single = nseg <= cap;
    if (single) {
      cache.load(src, i, sb, (int)nseg, threadIdx.x, THREADS);
      __syncthreads();
      if (preall) {
        const int lane = threadIdx.x & 31, n = (int)nseg;
        for (int p = threadIdx.x >> 5; p < npanels; p += NW) {
          int* pp = pre_all + (size_t)p * (cap + 1);
          int run = 0;
          for (int t0 = 0; t0 < n; t0 += 32) {
            const int ln = t0 + lane < n ? cache.len(t0 + lane, p) : 0;
            int incl = ln;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
              const int x = __shfl_up_sync(kFull, incl, d);
              if (lane >= d) incl += x;
            }
            if (t0 + lane < n) pp[t0 + lane] = run + incl - ln;
            run += __shfl_sync(kFull, incl, 31);
          }
          if (lane == 0) pp[n] = run;
        }
        __syncthreads();
      }
    }
    int64_t written = 0;
    if (threadIdx.x == 0 && out.bump) out.rowstart[i] = -2;  // chunked: see out.chunks
    for (int p = 0; p < npanels; ++p) {
      const int lo = p * W;
      for (int64_t c0 = 0; c0 < nseg; c0 += cap) {
        const int n = (int)(nseg - c0 < (int64_t)cap ? nseg - c0 : (int64_t)cap);
        if (!single) {
          cache.load(src, i, sb + c0, n, threadIdx.x, THREADS);
          __syncthreads();
        }
        if (preall && single) {
          cache.pre = pre_all + (size_t)p * (cap + 1);
        } else {
          cache.pre = pre0;
          cache.template prefix<THREADS, Count>(n, p, scan_tmp);
        }
#ifdef SPG_ABL_NO_ATOMIC  // ablation build: loads and products only
        balanced_items<SR, Src, NW, kDenseIPL>(src, cache, n, p, [&](int32_t c, const V& v) {
          if (bits_equal(v, SR::one()) && c == -7) acc[0] = v;
        });
#else
        balanced_items<SR, Src, NW, kDenseIPL, false, true>(src, cache, n, p, [&](int32_t c, const V& v) {
          if (SR::is_zero(v)) return;  // add(x, zero) == x: nothing to fold
          const int cc = c - lo;
          const V old = atomic_accumulate<SR, true>(&acc[cc], v);
          if (is_zero_bits<SR>(old)) atomicOr(&bm[cc >> 5], 1u << (cc & 31));  // first touch
        });
#endif
        __syncthreads();
      }
#ifdef SPG_ABL_NO_EMIT  // ablation build: clear instead of emitting
      for (int e = threadIdx.x; e < W / 32; e += THREADS)
        if (bm[e]) {
          for (uint32_t y = bm[e]; y; y &= y - 1) acc[(e << 5) + __ffs(y) - 1] = SR::zero();
          bm[e] = 0u;
        }
      __syncthreads();
#else
      if (warp_emit) {
        bitmap_emit_warp<SR, W, THREADS>(acc, bm, lo, out, i, r, p, &s_fill);
        __syncthreads();  // slices cleared before the next panel's atomics
      } else {
        written += bitmap_emit<SR, W, THREADS>(acc, bm, lo, out, i, r, p, npanels, written, wsum, &s_base);
      }
#endif
    }
    if (threadIdx.x == 0) out.rownnz[i] = warp_emit ? s_fill : written;
  }
}

// ---------------------------------------------------------------------------
// K5' bin 6, warp-specialised: PW product warps fold panel p into one of two
// accumulators while EW emit warps write out panel p-1 from the other, so
// the ordered emission overlaps the next panel's gathers and atomics.
// Hand-off per accumulator buffer b through named barriers:
//   FULL(b) = 1 + b : product warps arrive after folding, emit warps sync;
//   FREE(b) = 3 + b : emit warps arrive after emitting, product warps sync.
// Barrier 5 = product warps only (segment-cache reload, prefix scan),
// barrier 6 = emit warps only (inside bitmap_emit).
// ---------------------------------------------------------------------------
template <class SR, class Src, int W, int PW, int EW>
__global__ void __launch_bounds__((PW + EW) * 32, 1) dense_panel_ws_kernel(Src src, const int64_t* __restrict__ rows,
                                                                          int64_t nrows_bin, int npanels, int cap,
                                                                          unsigned long long* __restrict__ work,
                                                                          RowOut<typename SR::value_type> out) {
  using V = typename SR::value_type;
  constexpr int NT = (PW + EW) * 32, PT = PW * 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* acc = reinterpret_cast<V*>(smem_raw);                               // [2][W]
  uint32_t* bm = reinterpret_cast<uint32_t*>(smem_raw + 2 * sizeof(V) * W);  // [2][W/32]
  SegCache<SR, Src> cache;
  cache.carve(smem_raw + 2 * sizeof(V) * W + 2 * sizeof(uint32_t) * (W / 32), cap, npanels);
  __shared__ long long s_row, s_base;
  __shared__ int wsum[2 * EW + 1];
  __shared__ int psum[PW + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool producer = warp < PW;

  for (int e = threadIdx.x; e < 2 * W; e += NT) acc[e] = SR::zero();
  for (int e = threadIdx.x; e < 2 * (W / 32); e += NT) bm[e] = 0u;
  __syncthreads();
  if (!producer) {  // both buffers start free
    named_arrive(3, NT);
    named_arrive(4, NT);
  }
  unsigned gp = 0;  // panels handed off so far (selects the buffer)
  for (;;) {
    if (threadIdx.x == 0) {
      const unsigned long long r = atomicAdd(work, 1ull);
      s_row = r < (unsigned long long)nrows_bin ? (long long)r : -1;
    }
    __syncthreads();  // previous row fully emitted; s_row visible
    const long long r = s_row;
    if (r < 0) break;
    const int64_t i = rows[r];
    const int64_t sb = src.seg_begin(i), se = src.seg_end(i);
    const int64_t nseg = se - sb;
    const bool single = nseg <= cap;
    if (single) {
      cache.load(src, i, sb, (int)nseg, threadIdx.x, NT);
      __syncthreads();
    }
    if (producer) {
      for (int p = 0; p < npanels; ++p, ++gp) {
        const int b = gp & 1;
        named_sync(3 + b, NT);  // buffer b emitted and cleared
        V* a = acc + b * W;
        uint32_t* m = bm + b * (W / 32);
        const int lo = p * W;
        for (int64_t c0 = 0; c0 < nseg; c0 += cap) {
          const int n = (int)(nseg - c0 < (int64_t)cap ? nseg - c0 : (int64_t)cap);
          if (!single) {
            named_sync(5, PT);  // previous batch's items consumed
            cache.load(src, i, sb + c0, n, threadIdx.x, PT);
            named_sync(5, PT);
          }
          // pre[0..n] = prefix of the panel-p slice lengths (product warps)
          {
            const int ipt = (n + PT - 1) / PT;
            const int t0 = threadIdx.x * ipt;
            int local = 0;
            for (int q = 0; q < ipt; ++q)
              if (t0 + q < n) local += cache.len(t0 + q, p);
            int incl = local;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
              const int x = __shfl_up_sync(kFull, incl, d);
              if (lane >= d) incl += x;
            }
            if (lane == 31) psum[warp] = incl;
            named_sync(5, PT);
            if (warp == 0) {
              const int v = lane < PW ? psum[lane] : 0;
              int wi = v;
#pragma unroll
              for (int d = 1; d < 32; d <<= 1) {
                const int x = __shfl_up_sync(kFull, wi, d);
                if (lane >= d) wi += x;
              }
              if (lane < PW) psum[lane] = wi - v;
              if (lane == 31) psum[PW] = wi;
            }
            named_sync(5, PT);
            int first = psum[warp] + incl - local;
            for (int q = 0; q < ipt; ++q)
              if (t0 + q < n) {
                cache.pre[t0 + q] = first;
                first += cache.len(t0 + q, p);
              }
            if (threadIdx.x == 0) cache.pre[n] = psum[PW];
            named_sync(5, PT);
          }
          balanced_items<SR, Src, PW, kDenseIPL>(src, cache, n, p, [&](int32_t c, const V& v) {
            if (SR::is_zero(v)) return;
            const int cc = c - lo;
            const V old = atomic_accumulate<SR, true>(&a[cc], v);
            if (is_zero_bits<SR>(old)) atomicOr(&m[cc >> 5], 1u << (cc & 31));
          });
          if (!single) named_sync(5, PT);
        }
        __threadfence_block();
        named_arrive(1 + b, NT);  // panel p ready for emission
      }
    } else {
      int64_t written = 0;
      for (int p = 0; p < npanels; ++p, ++gp) {
        const int b = gp & 1;
        named_sync(1 + b, NT);  // panel p folded
        written += bitmap_emit<SR, W, EW * 32, 6, PW>(acc + b * W, bm + b * (W / 32), p * W, out, i, r, p, npanels,
                                                       written, wsum, &s_base);
        named_arrive(3 + b, NT);  // buffer b free again
      }
      if (threadIdx.x == PT) {
        out.rownnz[i] = written;
        if (out.bump) out.rowstart[i] = -2;
      }
    }
  }
  if (producer) {  // consume the last two FREE hand-offs
    named_sync(3, NT);
    named_sync(4, NT);
  }
}

// ---------------------------------------------------------------------------
// K4' bin 8: bit-rank accumulator for mid-size rows whose output columns lie
// in a window [colmin, colmin + span) of at most 32*WMAX columns.  Pass 1
// sets a presence bit per product column (plus a summary bit per non-empty
// word); the non-empty words, listed in order from the summary, get their
// word ranks by one block scan, so every present column's rank is its output
// position; pass 2 folds each product into acc[rank] with native smem
// atomics; the output is the bitmap expanded in order plus acc[0..nnz)
// copied straight out — sorted without sorting, no probing, no column
// panels, and per-row work proportional to the non-empty words only.
// Not used for semirings whose fold can cancel to zero (fp64 +).
// ---------------------------------------------------------------------------
template <class SR, class Src, int THREADS, int NMAX, int WMAX>
__global__ void __launch_bounds__(THREADS) bitrank_rows_kernel(Src src, const int64_t* __restrict__ rows,
                                                               int64_t nrows_bin, int cap,
                                                               const int32_t* __restrict__ colmin,
                                                               RowOut<typename SR::value_type> out) {
  using V = typename SR::value_type;
  constexpr int NW = THREADS / 32;
  constexpr int SW = WMAX / 32;                        // summary words
  static_assert(NMAX <= 65535 && WMAX <= 65536 && SW <= THREADS, "bit-rank geometry");
  constexpr int LPT0 = (NMAX + THREADS - 1) / THREADS;
  constexpr int LPT = LPT0 >= 16 ? (LPT0 | 1) : LPT0;  // listed words per thread (odd when long: fewer bank conflicts)
  using Scan = cub::BlockScan<int, THREADS>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* acc = reinterpret_cast<V*>(smem_raw);                               // [NMAX]
  uint32_t* bm = reinterpret_cast<uint32_t*>(acc + NMAX);                // [WMAX] presence
  uint32_t* sm = bm + WMAX;                                              // [SW] non-empty words
  uint16_t* wrank = reinterpret_cast<uint16_t*>(sm + SW);                // [WMAX] rank of a word's first entry
  constexpr int LMAX = NMAX < WMAX ? NMAX : WMAX;                        // non-empty words <= both
  uint16_t* list = wrank + WMAX;                                         // [LMAX] non-empty words in order
  SegCache<SR, Src> cache;
  cache.carve(reinterpret_cast<unsigned char*>(list + ((LMAX + 7) & ~7)), cap, 1);
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ long long s_base;
  __shared__ int s_nw;
  for (int e = threadIdx.x; e < WMAX; e += THREADS) bm[e] = 0u;
  for (int e = threadIdx.x; e < SW; e += THREADS) sm[e] = 0u;
  __syncthreads();
  for (int64_t r = blockIdx.x; r < nrows_bin; r += gridDim.x) {
    const int64_t i = rows[r];
    const int32_t lo = colmin[i];
    const int64_t sb = src.seg_begin(i);
    const int n = (int)(src.seg_end(i) - sb);  // <= cap by binning
    cache.load(src, i, sb, n, threadIdx.x, THREADS);
    __syncthreads();
    cache.template prefix<THREADS, Scan>(n, 0, scan_tmp);
    // pass 1: presence (+ summary bit on a word's first touch)
    balanced_items<SR, Src, NW>(src, cache, n, 0, [&](int32_t c, const V& v) {
      if (SR::is_zero(v)) return;
      const int cc = c - lo, w = cc >> 5;
      if (atomicOr(&bm[w], 1u << (cc & 31)) == 0u) atomicOr(&sm[w >> 5], 1u << (w & 31));
    });
    __syncthreads();
    // list the non-empty words in order (summary word t -> thread t)
    {
      const uint32_t x = threadIdx.x < SW ? sm[threadIdx.x] : 0u;
      int first, nw;
      Scan(scan_tmp).ExclusiveSum(__popc(x), first, nw);
      for (uint32_t y = x; y; y &= y - 1) list[first++] = (uint16_t)((threadIdx.x << 5) + __ffs(y) - 1);
      if (threadIdx.x == 0) s_nw = nw;
    }
    __syncthreads();
    const int nw = s_nw;
    // word ranks: block scan of the popcounts over the listed words (blocked)
    int local = 0;
    const int k0 = threadIdx.x * LPT;
#pragma unroll
    for (int q = 0; q < LPT; ++q)
      if (k0 + q < nw) local += __popc(bm[list[k0 + q]]);
    int first, total;
    Scan(scan_tmp).ExclusiveSum(local, first, total);
#pragma unroll
    for (int q = 0; q < LPT; ++q)
      if (k0 + q < nw) {
        const int w = list[k0 + q];
        wrank[w] = (uint16_t)first;
        first += __popc(bm[w]);
      }
    for (int e = threadIdx.x; e < total; e += THREADS) acc[e] = SR::zero();
    __syncthreads();
    // pass 2: fold into acc[rank]
    balanced_items<SR, Src, NW>(src, cache, n, 0, [&](int32_t c, const V& v) {
      if (SR::is_zero(v)) return;
      const int cc = c - lo, w = cc >> 5;
      atomic_accumulate<SR, true>(&acc[wrank[w] + __popc(bm[w] & ((1u << (cc & 31)) - 1u))], v);
    });
    __syncthreads();
    if (threadIdx.x == 0) {
      s_base = out.claim_row(i, total);
      out.rownnz[i] = total;
    }
    __syncthreads();
    // emit: columns expanded from the listed words, values straight from acc
    const int64_t o = s_base;
    if (o >= 0) {
      // striped over the listed words: neighbouring lanes write neighbouring output runs
      for (int kw = threadIdx.x; kw < nw; kw += THREADS) {
          const int w = list[kw];
          int k = wrank[w];
          for (uint32_t y = bm[w]; y; y &= y - 1) out.cols[o + k++] = lo + (w << 5) + __ffs(y) - 1;
        }
      for (int e = threadIdx.x; e < total; e += THREADS) out.vals[o + e] = acc[e];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < LPT; ++q)
      if (k0 + q < nw) bm[list[k0 + q]] = 0u;
    if (threadIdx.x < SW) sm[threadIdx.x] = 0u;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K5'' bin 9: rank panels.  Long rows whose output columns fit a window of
// 32*WMAX columns: pass 1 marks presence over the whole window, a block scan
// of the non-empty words' popcounts ranks every output column (= its output
// position), all output columns are written at once, and the values are
// folded panel by panel in RANK space — panel k holds ranks [k*NMAX,
// (k+1)*NMAX), i.e. a column range found from the ranks, so every
// accumulator slot is an output and a row needs ceil(nnz/NMAX) panels
// instead of ncols/W.  Segment slices per panel come from binary searches
// in the (sorted) right-operand rows.  Emission is a contiguous copy.
// ---------------------------------------------------------------------------
template <class SR, class Src, int THREADS, int NMAX, int WMAX>
__global__ void __launch_bounds__(THREADS, THREADS <= 512 ? 2 : 1) rankpanel_rows_kernel(Src src, const int64_t* __restrict__ rows,
                                                                    int64_t nrows_bin, int cap,
                                                                    const int32_t* __restrict__ colmin,
                                                                    RowOut<typename SR::value_type> out) {
  using V = typename SR::value_type;
  constexpr int NW = THREADS / 32;
  constexpr int SW = WMAX / 32;
  constexpr int LPT0 = (WMAX + THREADS - 1) / THREADS;
  constexpr int LPT = LPT0 >= 16 ? (LPT0 | 1) : LPT0;  // listed words per thread (odd when long: fewer bank conflicts)
  static_assert(WMAX <= 65536 && SW <= THREADS, "rank-panel geometry");
  using Scan = cub::BlockScan<int, THREADS>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* acc = reinterpret_cast<V*>(smem_raw);                  // [NMAX]
  uint32_t* bm = reinterpret_cast<uint32_t*>(acc + NMAX);   // [WMAX]
  uint32_t* sm = bm + WMAX;                                 // [SW]
  uint16_t* wrank = reinterpret_cast<uint16_t*>(sm + SW);   // [WMAX] (ranks < F <= 65535 by binning)
  uint16_t* list = wrank + WMAX;                            // [WMAX]
  int64_t* b0 = reinterpret_cast<int64_t*>(list + WMAX);    // [cap] whole-segment starts
  int* len0 = reinterpret_cast<int*>(b0 + cap);             // [cap]
  SegCache<SR, Src> cache;
  cache.carve(reinterpret_cast<unsigned char*>(len0 + ((cap + 3) & ~3)), cap, 1);
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ long long s_base;
  __shared__ int s_nw, s_clo, s_chi;
  for (int e = threadIdx.x; e < WMAX; e += THREADS) bm[e] = 0u;
  for (int e = threadIdx.x; e < SW; e += THREADS) sm[e] = 0u;
  __syncthreads();
  for (int64_t r = blockIdx.x; r < nrows_bin; r += gridDim.x) {
    const int64_t i = rows[r];
    const int32_t lo = colmin[i];
    const int64_t sb = src.seg_begin(i);
    const int n = (int)(src.seg_end(i) - sb);  // <= cap by binning
    cache.load(src, i, sb, n, threadIdx.x, THREADS);
    __syncthreads();
    for (int t = threadIdx.x; t < n; t += THREADS) {
      b0[t] = cache.b[t];
      len0[t] = cache.po[t];
    }
    cache.template prefix<THREADS, Scan>(n, 0, scan_tmp);
    // pass 1: presence over the window (+ summary bit on a word's first touch)
    balanced_items<SR, Src, NW>(src, cache, n, 0, [&](int32_t c, const V& v) {
      if (SR::is_zero(v)) return;
      const int cc = c - lo, w = cc >> 5;
      if (atomicOr(&bm[w], 1u << (cc & 31)) == 0u) atomicOr(&sm[w >> 5], 1u << (w & 31));
    });
    __syncthreads();
    {
      const uint32_t x = threadIdx.x < SW ? sm[threadIdx.x] : 0u;
      int first, nw;
      Scan(scan_tmp).ExclusiveSum(__popc(x), first, nw);
      for (uint32_t y = x; y; y &= y - 1) list[first++] = (uint16_t)((threadIdx.x << 5) + __ffs(y) - 1);
      if (threadIdx.x == 0) s_nw = nw;
    }
    __syncthreads();
    const int nw = s_nw;
    const int k0 = threadIdx.x * LPT;
    int local = 0;
#pragma unroll
    for (int q = 0; q < LPT; ++q)
      if (k0 + q < nw) local += __popc(bm[list[k0 + q]]);
    int first, total;
    Scan(scan_tmp).ExclusiveSum(local, first, total);
#pragma unroll
    for (int q = 0; q < LPT; ++q)
      if (k0 + q < nw) {
        const int w = list[k0 + q];
        wrank[w] = (uint16_t)first;
        first += __popc(bm[w]);
      }
    if (threadIdx.x == 0) {
      s_base = out.claim_row(i, total);
      out.rownnz[i] = total;
    }
    __syncthreads();
    const int64_t o = s_base;
    // all output columns of the row
    if (o >= 0) {
      // striped over the listed words: neighbouring lanes write neighbouring output runs
      for (int kw = threadIdx.x; kw < nw; kw += THREADS) {
          const int w = list[kw];
          int k = wrank[w];
          for (uint32_t y = bm[w]; y; y &= y - 1) out.cols[o + k++] = lo + (w << 5) + __ffs(y) - 1;
        }
    }
    const int npan = (total + NMAX - 1) / NMAX;
    for (int pk = 0; pk < npan; ++pk) {
      const int R0 = pk * NMAX, R1 = min(total, R0 + NMAX);
      if (npan > 1) {
        // window columns of ranks R0 and R1-1
#pragma unroll
        for (int q = 0; q < LPT; ++q)
          if (k0 + q < nw) {
            const int w = list[k0 + q];
            const int a = wrank[w], c = __popc(bm[w]);
            if (a <= R0 && R0 < a + c) s_clo = (w << 5) + nth_set_bit(bm[w], R0 - a);
            if (a <= R1 - 1 && R1 - 1 < a + c) s_chi = (w << 5) + nth_set_bit(bm[w], R1 - 1 - a);
          }
        __syncthreads();
        const int clo = lo + s_clo, chi = lo + s_chi;
        // each segment's slice with columns in [clo, chi] (binary searches in the sorted R row)
        for (int t = threadIdx.x; t < n; t += THREADS) {
          const int64_t bb = b0[t];
          const int sd = cache.sid[t];
          int a = 0, z = len0[t];  // first position with col >= clo
          while (a < z) {
            const int mid = (a + z) >> 1;
            if (src.col(sd, bb + mid) < clo) a = mid + 1;
            else z = mid;
          }
          int e = a, y = len0[t];  // first position with col > chi
          while (e < y) {
            const int mid = (e + y) >> 1;
            if (src.col(sd, bb + mid) <= chi) e = mid + 1;
            else y = mid;
          }
          cache.b[t] = bb + a;
          cache.po[t] = e - a;
        }
        __syncthreads();
        cache.template prefix<THREADS, Scan>(n, 0, scan_tmp);
      }
      for (int e = threadIdx.x; e < R1 - R0; e += THREADS) acc[e] = SR::zero();
      __syncthreads();
      balanced_items<SR, Src, NW>(src, cache, n, 0, [&](int32_t c, const V& v) {
        if (SR::is_zero(v)) return;
        const int cc = c - lo, w = cc >> 5;
        atomic_accumulate<SR, true>(&acc[wrank[w] + __popc(bm[w] & ((1u << (cc & 31)) - 1u)) - R0], v);
      });
      __syncthreads();
      if (o >= 0)
        for (int e = threadIdx.x; e < R1 - R0; e += THREADS) out.vals[o + R0 + e] = acc[e];
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < LPT; ++q)
      if (k0 + q < nw) bm[list[k0 + q]] = 0u;
    if (threadIdx.x < SW) sm[threadIdx.x] = 0u;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Shared-memory bitonic sort of n uint64 keys (pads to a power of two).
// ---------------------------------------------------------------------------
template <int THREADS>
__device__ __forceinline__ void block_bitonic_sort(uint64_t* buf, int n) {
  int p = 1, lp = 0;
  while (p < n) {
    p <<= 1;
    ++lp;
  }
  for (int e = n + threadIdx.x; e < p; e += THREADS) buf[e] = ~0ull;
  __syncthreads();
  for (int lk = 1; lk <= lp; ++lk) {
    for (int lj = lk - 1; lj >= 0; --lj) {
      const int j = 1 << lj;
      for (int t = threadIdx.x; t < (p >> 1); t += THREADS) {
        const int a = ((t >> lj) << (lj + 1)) | (t & (j - 1));
        const int b = a + j;
        const uint64_t x = buf[a], y = buf[b];
        const bool up = ((a >> lk) & 1) == 0;
        if ((x > y) == up) {
          buf[a] = y;
          buf[b] = x;
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ uint32_t hash_slot(uint32_t col, int log2t) {
  return (col * 2654435769u) >> (32 - log2t);
}

// ---------------------------------------------------------------------------
// K4 bins 3,4,7: CTA-wide shared-memory hash accumulator with T slots (load
// factor <= 1/2), balanced warp enumeration, compaction + bitonic sort of the
// occupied slots.  Used for medium rows and for outputs too wide for panels.
// ---------------------------------------------------------------------------
template <int T, int THREADS>
struct HashSort {
  using Scan = cub::BlockScan<int, THREADS>;
  union Tmp {
    typename Scan::TempStorage scan;
  };
};

// OPT (optimistic small table): rows are tried in a table sized for their
// likely distinct count; a row whose distinct columns pass T/2 stops
// inserting (at most THREADS more keys land, so probing always finds a free
// slot), writes nothing and is listed in ovf_rows for a re-run in a full-size
// table.  A stencil row (729 products, 125 outputs) then touches 512 slots
// instead of 2048, at 4x the CTAs per SM.
// GRED: the slot values live in a per-CTA table in global memory (gtab,
// zero on entry and left zero) and fold with acc_global (a native L2
// reduction for fp64 +, instead of a shared-memory CAS loop); after a row's
// fold its occupied slots are copied into shared memory and re-zeroed.
template <class SR, class Src, int T, int THREADS, bool OPT = false, bool GRED = false>
__global__ void __launch_bounds__(THREADS) hash_rows_kernel(Src src, const int64_t* __restrict__ rows,
                                                            int64_t nrows_bin, int cap, int end_bit,
                                                            RowOut<typename SR::value_type> out,
                                                            unsigned long long* ovf_n = nullptr,
                                                            int64_t* ovf_rows = nullptr,
                                                            typename SR::value_type* gtab = nullptr) {
  using V = typename SR::value_type;
  using HS = HashSort<T, THREADS>;
  __shared__ long long s_base;
  __shared__ int s_distinct, s_over;  // OPT only
  constexpr int SPT = T / THREADS;
  constexpr int NW = THREADS / 32;
  constexpr int NB = T / 2, NBT = NB / THREADS, kBucketMax = 32;
  static_assert(NB % THREADS == 0, "bucket count must divide by the CTA size");
  constexpr int LOG2T = (T == 512) ? 9 : (T == 1024) ? 10 : (T == 2048) ? 11 : (T == 4096) ? 12
                      : (T == 8192) ? 13 : (T == 16384) ? 14 : 15;
  static_assert((1 << LOG2T) == T, "T must be a power of two");
  static_assert(T <= 65536, "slot ids must fit 16 bits");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // layout: values [T] | keys [T] (later: bucket starts [T/2] + bucketed keys [T/2])
  //         | staging: keys [T/2] + (slot | rank << 16) [T/2] | cub temp | segment cache
  V* tvals = reinterpret_cast<V*>(smem_raw);
  int32_t* tkeys = reinterpret_cast<int32_t*>(smem_raw + sizeof(V) * T);
  uint32_t* stg_key = reinterpret_cast<uint32_t*>(tkeys + T);
  uint32_t* stg_slot = stg_key + T / 2;
  typename HS::Tmp* tmp = reinterpret_cast<typename HS::Tmp*>(stg_slot + T / 2);
  int* bstart = tkeys;                                        // after staging
  uint32_t* bkeys = reinterpret_cast<uint32_t*>(tkeys) + NB;  // after staging
  SegCache<SR, Src> cache;
  cache.carve(reinterpret_cast<unsigned char*>(tmp) + ((sizeof(typename HS::Tmp) + 15) & ~size_t(15)), cap, 1);
  const int shift = end_bit > LOG2T - 1 ? end_bit - (LOG2T - 1) : 0;
  V* gv = GRED ? gtab + (size_t)blockIdx.x * T : nullptr;
  for (int64_t r = blockIdx.x; r < nrows_bin; r += gridDim.x) {
    const int64_t i = rows[r];
    for (int e = threadIdx.x; e < T; e += THREADS) {
      tkeys[e] = kEmptyKey;
      if constexpr (!GRED) tvals[e] = SR::zero();
    }
    if (OPT && threadIdx.x == 0) {
      s_distinct = 0;
      s_over = 0;
    }
    const int64_t sb = src.seg_begin(i), nseg = src.seg_end(i) - sb;
    for (int64_t c0 = 0; c0 < nseg; c0 += cap) {
      const int n = (int)(nseg - c0 < (int64_t)cap ? nseg - c0 : (int64_t)cap);
      cache.load(src, i, sb + c0, n, threadIdx.x, THREADS);
      __syncthreads();
      cache.template prefix<THREADS, typename HS::Scan>(n, 0, tmp->scan);
      balanced_items<SR, Src, NW>(src, cache, n, 0, [&](int32_t c, const V& v) {
        if (SR::is_zero(v)) return;
        if constexpr (OPT) {
          if (*reinterpret_cast<volatile int*>(&s_over)) return;
        }
        uint32_t h = hash_slot((uint32_t)c, LOG2T);
        int probes = 0;
        for (;;) {
          const int32_t k = *reinterpret_cast<volatile int32_t*>(&tkeys[h]);
          if (k == c) break;
          if (k == kEmptyKey) {
            const int32_t prev = atomicCAS(&tkeys[h], kEmptyKey, c);
            if (prev == kEmptyKey) {
              if constexpr (OPT) {
                if (atomicAdd(&s_distinct, 1) >= T / 2) {
                  s_over = 1;
                  return;
                }
              }
              break;
            }
            if (prev == c) break;
          }
          h = (h + 1) & (T - 1);
          SPG_DCHECK(++probes < T);  // the bin keeps the table at most half full (OPT: < T/2 + THREADS keys)
        }
        if constexpr (GRED) {
          if constexpr (std::is_same<V, double>::value)  // fire-and-forget L2 reduction (no returned value)
            asm volatile("red.global.add.f64 [%0], %1;" ::"l"(gv + h), "d"(v) : "memory");
          else
            SR::acc_global(&gv[h], v);
        } else {
          atomic_accumulate<SR, true>(&tvals[h], v);
        }
      });
      if constexpr (GRED) __threadfence_block();  // the reductions land before any thread reads gv
      __syncthreads();
    }
    if constexpr (GRED) {  // occupied slots: value into shared memory, global slot back to zero
#pragma unroll 4
      for (int q = 0; q < SPT; ++q) {
        const int e = threadIdx.x + q * THREADS;
        if (tkeys[e] != kEmptyKey) {
          tvals[e] = gv[e];
          gv[e] = SR::zero();
        }
      }
      __threadfence_block();  // zeros visible before the next row's reductions (after the barriers below)
    }
    if constexpr (OPT) {
      if (s_over) {  // uniform after the barrier: re-run in the full-size table
        if (threadIdx.x == 0) ovf_rows[atomicAdd(ovf_n, 1ull)] = i;
        __syncthreads();
        continue;
      }
    }
    // occupied, non-zero slots -> staging.  Slots are taken striped (slot
    // t + q*THREADS: conflict-free shared loads); staging order is free, the
    // bucketing below sorts by column.
    int cnt = 0;
#pragma unroll 4
    for (int q = 0; q < SPT; ++q) {
      const int e = threadIdx.x + q * THREADS;
      cnt += (tkeys[e] != kEmptyKey && !SR::is_zero(tvals[e])) ? 1 : 0;
    }
    int first, total;
    typename HS::Scan(tmp->scan).ExclusiveSum(cnt, first, total);
    if (threadIdx.x == 0) {
      s_base = out.claim_row(i, total);
      out.rownnz[i] = total;
    }
    if (!out.writes()) {  // counting pass: no sort, no output
      __syncthreads();
      continue;
    }
#pragma unroll 4
    for (int q = 0; q < SPT; ++q) {
      const int e = threadIdx.x + q * THREADS;
      const int32_t k = tkeys[e];
      if (k != kEmptyKey && !SR::is_zero(tvals[e])) {
        stg_key[first] = (uint32_t)k;
        stg_slot[first] = (uint32_t)e;
        ++first;
      }
    }
    __syncthreads();  // the key table is free from here on
    const int64_t o = s_base;
    // Monotone bucketing by the high column bits: NB = T/2 buckets (>= the
    // entries), counts by shared atomics (the arrival rank rides in bits
    // 16..31 of the staged slot), starts by one block scan, in-bucket order
    // by a rank count; each entry is stored straight at its sorted position.
    // A row whose columns crowd one bucket (> kBucketMax) is radix-sorted.
    for (int b = threadIdx.x; b < NB; b += THREADS) bstart[b] = 0;
    __syncthreads();
    for (int e = threadIdx.x; e < total; e += THREADS)
      stg_slot[e] |= (uint32_t)min(atomicAdd(&bstart[stg_key[e] >> shift], 1), 0xffff) << 16;
    __syncthreads();
    int sum = 0, mx = 0;
#pragma unroll
    for (int b = 0; b < NBT; ++b) {
      const int n = bstart[threadIdx.x * NBT + b];
      sum += n;
      mx = max(mx, n);
    }
    if (!__syncthreads_or(mx > kBucketMax)) {
      int run;
      typename HS::Scan(tmp->scan).ExclusiveSum(sum, run);
#pragma unroll
      for (int b = 0; b < NBT; ++b) {
        const int n = bstart[threadIdx.x * NBT + b];
        bstart[threadIdx.x * NBT + b] = run;
        run += n;
      }
      __syncthreads();
      for (int e = threadIdx.x; e < total; e += THREADS)
        bkeys[bstart[stg_key[e] >> shift] + (stg_slot[e] >> 16)] = stg_key[e];
      __syncthreads();
      if (o >= 0)
        for (int e = threadIdx.x; e < total; e += THREADS) {
          const uint32_t key = stg_key[e];
          const int b = (int)(key >> shift);
          const int s1 = b + 1 < NB ? bstart[b + 1] : total;
          int pos = bstart[b];
          for (int j = pos; j < s1; ++j) pos += bkeys[j] < key;
          out.cols[o + pos] = (int32_t)key;
          out.vals[o + pos] = tvals[stg_slot[e] & 0xffff];
        }
      __syncthreads();
      continue;
    }
    // skewed row: bitonic sort of (key << 32 | slot) in the free key table
    uint64_t* buf = reinterpret_cast<uint64_t*>(tkeys);
    __syncthreads();
    for (int e = threadIdx.x; e < total; e += THREADS)
      buf[e] = ((uint64_t)stg_key[e] << 32) | (stg_slot[e] & 0xffffu);
    block_bitonic_sort<THREADS>(buf, total);
    if (o >= 0)
      for (int e = threadIdx.x; e < total; e += THREADS) {
        const uint64_t x = buf[e];
        out.cols[o + e] = (int32_t)(x >> 32);
        out.vals[o + e] = tvals[(uint32_t)x & 0xffffu];
      }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K7: compaction scratch -> exact CSR (warp per row, 4-way unrolled)
// ---------------------------------------------------------------------------
// U-slot mode, dense rows with per-warp chunks: CTA per row; one block scan
// over the row's chunk counts gives each chunk its place in C (chunk starts
// and counts staged in smem with it), then each warp copies two chunks per
// step with both chunks' loads in flight before the stores (coalesced within
// a chunk; chunks average ~150 entries).
#ifndef SPG_COMPACT_MINB
#define SPG_COMPACT_MINB 4  // min resident CTAs/SM for the compaction kernels, values <= 4 B (64 regs; 1 -> 4 saves 0.3 ms, 6 spills; wider values spill)
#endif
template <class V, int THREADS>
__global__ void __launch_bounds__(THREADS, sizeof(V) <= 4 ? SPG_COMPACT_MINB : 1) compact_wchunks_kernel(const int64_t* __restrict__ rows, int64_t nrows_bin,
                                                                  const int32_t* __restrict__ wchunks, int wstride,
                                                                  const int64_t* __restrict__ off,
                                                                  const int64_t* __restrict__ rowptr,
                                                                  const int32_t* __restrict__ sc_cols,
                                                                  const V* __restrict__ sc_vals,
                                                                  int32_t* __restrict__ cols, V* __restrict__ vals) {
  using Scan = cub::BlockScan<int, THREADS>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int spos[THREADS], sbeg[THREADS], scnt[THREADS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = THREADS / 32, E = 8;  // entries per lane held in registers per chunk
  for (int64_t r = blockIdx.x; r < nrows_bin; r += gridDim.x) {
    const int64_t i = rows[r];
    const int32_t* ch = wchunks + 2 * (r * wstride);
    const int64_t s0 = off[i];
    int64_t d0 = rowptr[i];
    for (int t0 = 0; t0 < wstride; t0 += THREADS) {
      const int k = t0 + threadIdx.x;
      const int2 bc = k < wstride ? reinterpret_cast<const int2*>(ch)[k] : make_int2(0, 0);
      int pos, total;
      Scan(tmp).ExclusiveSum(bc.y, pos, total);
      spos[threadIdx.x] = pos;
      sbeg[threadIdx.x] = bc.x;
      scnt[threadIdx.x] = bc.y;
      __syncthreads();
      const int nk = min(THREADS, wstride - t0);
      // two chunks per step: both chunks' loads are in flight before either's stores
      for (int kk = warp; kk < nk; kk += 2 * NW) {
        const int k2 = kk + NW;
        const int na = scnt[kk], nb = k2 < nk ? scnt[k2] : 0;
        if (na > 32 * E || nb > 32 * E) {  // long chunk: plain loop
          for (int h = 0; h < 2; ++h) {
            const int kc = h ? k2 : kk;
            const int n = h ? nb : na;
            if (n == 0) continue;
            const int64_t sa = s0 + sbeg[kc], da = d0 + spos[kc];
            for (int e = lane; e < n; e += 32) {
              cols[da + e] = sc_cols[sa + e];
              vals[da + e] = sc_vals[sa + e];
            }
          }
          continue;
        }
        const int64_t sa = s0 + sbeg[kk], da = d0 + spos[kk];
        const int64_t sb = nb ? s0 + sbeg[k2] : 0, db = nb ? d0 + spos[k2] : 0;
        int32_t ca[E], cb[E];
        V va[E], vb[E];
#pragma unroll
        for (int u = 0; u < E; ++u) {
          const int e = lane + 32 * u;
          if (e < na) {
            ca[u] = sc_cols[sa + e];
            va[u] = sc_vals[sa + e];
          }
          if (e < nb) {
            cb[u] = sc_cols[sb + e];
            vb[u] = sc_vals[sb + e];
          }
        }
#pragma unroll
        for (int u = 0; u < E; ++u) {
          const int e = lane + 32 * u;
          if (e < na) {
            cols[da + e] = ca[u];
            vals[da + e] = va[u];
          }
          if (e < nb) {
            cols[db + e] = cb[u];
            vals[db + e] = vb[u];
          }
        }
      }
      d0 += total;
      __syncthreads();
    }
  }
}

// Dense rows: concatenate their per-panel chunks (CTA per row).
template <class V>
__global__ void __launch_bounds__(256) compact_chunks_kernel(const int64_t* __restrict__ rows, int64_t nrows_bin,
                                                             int npanels, const int64_t* __restrict__ chunks,
                                                             const int64_t* __restrict__ rowptr,
                                                             const int32_t* __restrict__ sc_cols,
                                                             const V* __restrict__ sc_vals, int32_t* __restrict__ cols,
                                                             V* __restrict__ vals) {
  for (int64_t r = blockIdx.x; r < nrows_bin; r += gridDim.x) {
    int64_t d = rowptr[rows[r]];
    for (int p = 0; p < npanels; ++p) {
      const int64_t s = chunks[2 * (r * npanels + p)], n = chunks[2 * (r * npanels + p) + 1];
      for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
        cols[d + e] = sc_cols[s + e];
        vals[d + e] = sc_vals[s + e];
      }
      d += n;
    }
  }
}

// Cooperative copy (threads tid of nt) of n 32-bit words from a 16-byte
// aligned source to any destination offset: aligned 16-byte stores, each
// output quad composed from two aligned source quads (the source may be read
// up to 3 words past n: scratch buffers carry slack).
__device__ __forceinline__ void copy_words(uint32_t* __restrict__ dst, int64_t d, const uint32_t* __restrict__ src,
                                           int64_t s, int64_t n, int tid, int nt) {
  const int64_t head = std::min<int64_t>((4 - (d & 3)) & 3, n);
  if (tid < head) dst[d + tid] = src[s + tid];
  const int64_t rest = n - head;
  if (rest <= 0) return;
  const int64_t nq = rest >> 2;
  const int64_t j0 = s + head;  // first source word of the aligned destination part
  const int sh = (int)(j0 & 3);
  const uint4* sq = reinterpret_cast<const uint4*>(src + (j0 - sh));
  uint4* dq = reinterpret_cast<uint4*>(dst + d + head);
  auto compose = [sh](const uint4& a, const uint4& b) {
    if (sh == 0) return a;
    if (sh == 1) return make_uint4(a.y, a.z, a.w, b.x);
    if (sh == 2) return make_uint4(a.z, a.w, b.x, b.y);
    return make_uint4(a.w, b.x, b.y, b.z);
  };
  constexpr int U = 4;  // quads in flight per thread
  int64_t k = tid;
  for (; k + (int64_t)nt * (U - 1) < nq; k += (int64_t)nt * U) {
    uint4 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      a[u] = __ldg(sq + k + (int64_t)nt * u);
      b[u] = sh ? __ldg(sq + k + (int64_t)nt * u + 1) : a[u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) dq[k + (int64_t)nt * u] = compose(a[u], b[u]);
  }
  for (; k < nq; k += nt) dq[k] = compose(__ldg(sq + k), sh ? __ldg(sq + k + 1) : make_uint4(0, 0, 0, 0));
  const int64_t t0 = head + (nq << 2);
  if (tid < n - t0) dst[d + t0 + tid] = src[s + t0 + tid];
}

// U-slot mode, dense rows (the long outputs): one CTA per row, 16-byte copies.
template <class V>
__global__ void __launch_bounds__(256) compact_long_rows_kernel(const int64_t* __restrict__ rows, int64_t nrows_bin,
                                                                const int64_t* __restrict__ off,
                                                                const int64_t* __restrict__ rowptr,
                                                                const int32_t* __restrict__ sc_cols,
                                                                const V* __restrict__ sc_vals,
                                                                int32_t* __restrict__ cols, V* __restrict__ vals) {
  static_assert(sizeof(V) % 4 == 0, "word copies need 4-byte multiples");
  constexpr int WPE = (int)(sizeof(V) / 4);
  for (int64_t r = blockIdx.x; r < nrows_bin; r += gridDim.x) {
    const int64_t i = rows[r];
    const int64_t d = rowptr[i], n = rowptr[i + 1] - d, s = off[i];
    copy_words(reinterpret_cast<uint32_t*>(cols), d, reinterpret_cast<const uint32_t*>(sc_cols), s, n, threadIdx.x,
               blockDim.x);
    copy_words(reinterpret_cast<uint32_t*>(vals), d * WPE, reinterpret_cast<const uint32_t*>(sc_vals), s * WPE,
               n * WPE, threadIdx.x, blockDim.x);
  }
}

#ifndef SPG_ROWS_VEC
#define SPG_ROWS_VEC 512  // rows with at least this many entries copy with 16-byte accesses (0: never)
#endif
// Other rows: row i sits at off[i] of the scratch (off[i] < 0: skip; rows
// whose bin is dense are skipped when `skip` is given).
template <class V>
__global__ void __launch_bounds__(256, sizeof(V) <= 4 ? SPG_COMPACT_MINB : 1) compact_rows_kernel(int64_t nrows, const uint8_t* __restrict__ skip,
                                                           const int64_t* __restrict__ off,
                                                           const int64_t* __restrict__ rowptr,
                                                           const int32_t* __restrict__ sc_cols,
                                                           const V* __restrict__ sc_vals, int32_t* __restrict__ cols,
                                                           V* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nrows; i += nwarps) {
    const int64_t d = rowptr[i];
    const int64_t n = rowptr[i + 1] - d;
    if (n == 0) continue;
    const int64_t s = off[i];
    if (s < 0) continue;
    if (skip && (skip[i] == kBinDense || skip[i] == kBinBitmap)) continue;  // copied by compact_long_rows_kernel
    if constexpr (SPG_ROWS_VEC > 0 && sizeof(V) % 4 == 0) {
      if (n >= SPG_ROWS_VEC) {  // long row: 16-byte loads and stores
        constexpr int WPE = (int)(sizeof(V) / 4);
        copy_words(reinterpret_cast<uint32_t*>(cols), d, reinterpret_cast<const uint32_t*>(sc_cols), s, n, lane, 32);
        copy_words(reinterpret_cast<uint32_t*>(vals), d * WPE, reinterpret_cast<const uint32_t*>(sc_vals), s * WPE,
                   n * WPE, lane, 32);
        continue;
      }
    }
    int64_t e = lane;
    for (; e + 96 < n; e += 128) {
      const int32_t c0 = sc_cols[s + e], c1 = sc_cols[s + e + 32], c2 = sc_cols[s + e + 64],
                    c3 = sc_cols[s + e + 96];
      const V v0 = sc_vals[s + e], v1 = sc_vals[s + e + 32], v2 = sc_vals[s + e + 64], v3 = sc_vals[s + e + 96];
      cols[d + e] = c0;
      cols[d + e + 32] = c1;
      cols[d + e + 64] = c2;
      cols[d + e + 96] = c3;
      vals[d + e] = v0;
      vals[d + e + 32] = v1;
      vals[d + e + 64] = v2;
      vals[d + e + 96] = v3;
    }
    for (; e < n; e += 32) {
      cols[d + e] = sc_cols[s + e];
      vals[d + e] = sc_vals[s + e];
    }
  }
}

}  // namespace spg
