// Row-accumulation kernels shared by the local multiply (esc_multiply
// replacement, local_spgemm.hpp:83-156) and the partial merge
// (merge_partials replacement, summa.hpp:122-172).
//
// Both operations have the same shape: output row i is the semiring fold of
// a list of SEGMENTS, each a sorted run of (column, value) items from some
// CSR row, optionally multiplied on the left by a scalar:
//   local multiply:  segments of row i = rows k of R for each A entry (i, k),
//                    item = mul(a_ik, r_kj)                     (Gustavson)
//   merge:           segments of row i = row i of each partial, item = value
// (the merge is the product [I I .. I] * vstack(partials)).  A Source type
// describes the segments; the kernels below are written once against it.
//
// Pipeline (one call):
//   K1 analyse   : per-row product count F_i, bound U_i = min(F_i, ncols),
//                  bin id                                    (warp per row)
//   K2 bin       : scatter rows into per-bin lists            (smem histogram)
//   K4 numeric   : per bin
//        bin 1  F_i <= 32   warp-ESC: products in registers, 32-lane bitonic
//                           sort on (col, product#), segmented shuffle fold
//        bin 2-5 U_i <= T/2 CTA hash table of T slots in shared memory
//                           (T = 512 .. 16K), atomic semiring accumulate,
//                           compaction + shared-memory bitonic sort
//        bin 6  larger      dense accumulator in global memory (L2-resident
//                           per-CTA slab) + bitmap; bitmap scan gives sorted
//                           output with no sort
//      each row writes into a scratch slot of U_i entries and reports nnz_i
//   K7 compact   : rowptr = scan(nnz); copy scratch -> exact-size CSR
#pragma once
#include <cub/block/block_scan.cuh>

#include "common.cuh"
#include "semiring.cuh"

namespace spg {

constexpr int kNumBins = 7;
constexpr int32_t kEmptyKey = -1;

// ---------------------------------------------------------------------------
// Sources
// ---------------------------------------------------------------------------
template <class SR>
struct MulSource {
  using V = typename SR::value_type;
  const int64_t* lptr;
  const int32_t* lidx;
  const V* lval;
  const int64_t* rptr;
  const int32_t* ridx;
  const V* rval;
  int64_t nrows;

  __device__ __forceinline__ int64_t seg_begin(int64_t i) const { return lptr[i]; }
  __device__ __forceinline__ int64_t seg_end(int64_t i) const { return lptr[i + 1]; }
  // Segment s of row i: R row lidx[s], scaled by lval[s].
  __device__ __forceinline__ void segment(int64_t /*i*/, int64_t s, int64_t& b, int64_t& len,
                                          const int32_t*& cols, const V*& vals, V& mult) const {
    const int32_t k = __ldg(lidx + s);
    b = __ldg(rptr + k);
    len = __ldg(rptr + k + 1) - b;
    cols = ridx;
    vals = rval;
    mult = lval[s];
  }
  __device__ __forceinline__ int64_t seg_len(int64_t /*i*/, int64_t s) const {
    const int32_t k = __ldg(lidx + s);
    return __ldg(rptr + k + 1) - __ldg(rptr + k);
  }
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
  MergeParts p;
  int nparts;
  int64_t nrows;

  __device__ __forceinline__ int64_t seg_begin(int64_t) const { return 0; }
  __device__ __forceinline__ int64_t seg_end(int64_t) const { return nparts; }
  __device__ __forceinline__ void segment(int64_t i, int64_t s, int64_t& b, int64_t& len,
                                          const int32_t*& cols, const V*& vals, V& mult) const {
    const int64_t* ptr = p.ptr[s];
    b = ptr[i];
    len = ptr[i + 1] - b;
    cols = p.idx[s];
    vals = static_cast<const V*>(p.val[s]);
    mult = SR::one();
  }
  __device__ __forceinline__ int64_t seg_len(int64_t i, int64_t s) const {
    const int64_t* ptr = p.ptr[s];
    return ptr[i + 1] - ptr[i];
  }
  __device__ __forceinline__ V item(const V&, const V& v) const { return v; }
};

template <class SR>
inline void rebase_source(MulSource<SR>& s, int64_t r0) {
  s.lptr += r0;
  s.nrows -= r0;
}
template <class SR>
inline void rebase_source(MergeSource<SR>& s, int64_t r0) {
  for (int q = 0; q < s.nparts; ++q) s.p.ptr[q] += r0;
  s.nrows -= r0;
}

// ---------------------------------------------------------------------------
// Bin geometry per value width
// ---------------------------------------------------------------------------
template <class V>
struct HashGeom {
  // largest table whose keys + values fit comfortably in 227 KB of smem
  static constexpr int kMaxT = sizeof(V) <= 1 ? 32768 : (sizeof(V) <= 8 ? 16384 : 8192);
};

// Table size for bins 2..5.
template <class V>
__host__ __device__ constexpr int bin_table(int bin) {
  return bin == 2 ? 512 : bin == 3 ? 2048 : bin == 4 ? 8192 : HashGeom<V>::kMaxT;
}

// ---------------------------------------------------------------------------
// K1: per-row analysis
// ---------------------------------------------------------------------------
template <class SR, class Src>
__global__ void __launch_bounds__(256) analyse_rows_kernel(Src src, int64_t ncols_out,
                                                           int64_t* __restrict__ prods,
                                                           int64_t* __restrict__ ubound,
                                                           uint8_t* __restrict__ bins) {
  using V = typename SR::value_type;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < src.nrows; i += nwarps) {
    const int64_t sb = src.seg_begin(i), se = src.seg_end(i);
    int64_t f = 0;
    for (int64_t s = sb + lane; s < se; s += 32) f += src.seg_len(i, s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
    if (lane == 0) {
      const int64_t u = f < ncols_out ? f : ncols_out;
      uint8_t b;
      if (f == 0) b = 0;
      else if (f <= 32) b = 1;
      else if (u <= bin_table<V>(2) / 2) b = 2;
      else if (u <= bin_table<V>(3) / 2) b = 3;
      else if (u <= bin_table<V>(4) / 2) b = 4;
      else if (u <= bin_table<V>(5) / 2) b = 5;
      else b = 6;
      prods[i] = f;
      ubound[i] = (b == 0) ? 0 : u;
      bins[i] = b;
    }
  }
}

// ---------------------------------------------------------------------------
// K2: bin scatter.  counts[b] must be zero on entry; lists are laid out at
// bin_base[b] (host-computed from a first counting launch).
// ---------------------------------------------------------------------------
static __global__ void __launch_bounds__(1024) bin_count_kernel(const uint8_t* __restrict__ bins,
                                                          int64_t n, unsigned long long* counts) {
  __shared__ unsigned int h[kNumBins];
  if (threadIdx.x < kNumBins) h[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&h[bins[i]], 1u);
  __syncthreads();
  if (threadIdx.x < kNumBins && h[threadIdx.x]) atomicAdd(&counts[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}

static __global__ void __launch_bounds__(1024) bin_scatter_kernel(const uint8_t* __restrict__ bins,
                                                            int64_t n,
                                                            unsigned long long* cursor,  // per bin, starts at base
                                                            int64_t* __restrict__ lists) {
  __shared__ unsigned int h[kNumBins];
  __shared__ unsigned long long base[kNumBins];
  const int64_t chunk0 = blockIdx.x * (int64_t)blockDim.x;
  for (int64_t c = chunk0; c < n; c += (int64_t)gridDim.x * blockDim.x) {
    if (threadIdx.x < kNumBins) h[threadIdx.x] = 0;
    __syncthreads();
    const int64_t i = c + threadIdx.x;
    int b = -1;
    unsigned int slot = 0;
    if (i < n) {
      b = bins[i];
      if (b != 0) slot = atomicAdd(&h[b], 1u);
    }
    __syncthreads();
    if (threadIdx.x < kNumBins) base[threadIdx.x] = h[threadIdx.x] ? atomicAdd(&cursor[threadIdx.x], (unsigned long long)h[threadIdx.x]) : 0;
    __syncthreads();
    if (b > 0) lists[base[b] + slot] = i;
    __syncthreads();
  }
}

static __global__ void zero_empty_rows_kernel(const uint8_t* __restrict__ bins, int64_t n,
                                       int64_t* __restrict__ rownnz) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (bins[i] == 0) rownnz[i] = 0;
}

// ---------------------------------------------------------------------------
// Value shuffles (any width)
// ---------------------------------------------------------------------------
template <class V>
__device__ __forceinline__ V shfl_v(const V& v, int src, unsigned mask = 0xffffffffu) {
  constexpr int W = (sizeof(V) + 3) / 4;
  uint32_t w[W];
  V out;
  memcpy(w, &v, sizeof(V) <= 4 * W ? sizeof(V) : 0);
  if constexpr (sizeof(V) < 4) w[0] = (uint32_t)(*reinterpret_cast<const uint8_t*>(&v));
#pragma unroll
  for (int k = 0; k < W; ++k) w[k] = __shfl_sync(mask, w[k], src);
  if constexpr (sizeof(V) < 4) {
    *reinterpret_cast<uint8_t*>(&out) = (uint8_t)w[0];
  } else {
    memcpy(&out, w, sizeof(V));
  }
  return out;
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
// K4 bin 1: warp-ESC for rows with <= 32 products
// ---------------------------------------------------------------------------
template <class SR, class Src>
__global__ void __launch_bounds__(256) esc_warp_kernel(Src src, const int64_t* __restrict__ rows,
                                                       int64_t nrows_bin,
                                                       const int64_t* __restrict__ off,
                                                       int32_t* __restrict__ out_cols,
                                                       typename SR::value_type* __restrict__ out_vals,
                                                       int64_t* __restrict__ rownnz) {
  using V = typename SR::value_type;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < nrows_bin; r += nwarps) {
    const int64_t i = rows[r];
    uint64_t key = ~0ull;  // (col << 32) | product#  ; ~0 = no item
    V val = SR::zero();
    int base = 0;
    const int64_t se = src.seg_end(i);
    for (int64_t s = src.seg_begin(i); s < se && base < 32; ++s) {
      int64_t b, len;
      const int32_t* cols;
      const V* vals;
      V mult;
      src.segment(i, s, b, len, cols, vals, mult);
      if (lane >= base && lane < base + len) {
        const int64_t u = b + (lane - base);
        key = ((uint64_t)(uint32_t)cols[u] << 32) | (uint32_t)lane;
        val = src.item(mult, vals[u]);
      }
      base += (int)len;
    }
    // 32-lane bitonic sort by key (unique keys -> deterministic fold order)
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        const uint64_t okey = __shfl_xor_sync(0xffffffffu, key, j);
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
    // segmented inclusive fold over equal columns
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t ocol = __shfl_up_sync(0xffffffffu, col, d);
      const V oval = shfl_up_v(val, d);
      if (lane >= d && ocol == col) val = SR::add(oval, val);
    }
    const uint32_t ncol = __shfl_down_sync(0xffffffffu, col, 1);
    const bool tail = valid && (lane == 31 || ncol != col);
    const bool keep = tail && !SR::is_zero(val);
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    const int pos = __popc(m & ((1u << lane) - 1));
    const int64_t o = off[i];
    if (keep) {
      out_cols[o + pos] = (int32_t)col;
      out_vals[o + pos] = val;
    }
    if (lane == 0) rownnz[i] = __popc(m);
  }
}

// ---------------------------------------------------------------------------
// Shared-memory bitonic sort of n uint64 keys (pads to a power of two).
// ---------------------------------------------------------------------------
template <int THREADS>
__device__ __forceinline__ void block_bitonic_sort(uint64_t* buf, int n) {
  int p = 1;
  while (p < n) p <<= 1;
  for (int e = n + threadIdx.x; e < p; e += THREADS) buf[e] = ~0ull;
  __syncthreads();
  for (int k = 2; k <= p; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < (p >> 1); t += THREADS) {
        const int a = 2 * j * (t / j) + (t % j);
        const int b = a + j;
        const uint64_t x = buf[a], y = buf[b];
        const bool up = (a & k) == 0;
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
// K4 bins 2-5: CTA-wide shared-memory hash accumulator, T slots.
// ---------------------------------------------------------------------------
template <class SR, class Src, int T, int THREADS>
__global__ void __launch_bounds__(THREADS) hash_rows_kernel(Src src, const int64_t* __restrict__ rows,
                                                            int64_t nrows_bin,
                                                            const int64_t* __restrict__ off,
                                                            int32_t* __restrict__ out_cols,
                                                            typename SR::value_type* __restrict__ out_vals,
                                                            int64_t* __restrict__ rownnz) {
  using V = typename SR::value_type;
  constexpr int SPT = T / THREADS;  // slots per thread in compaction
  constexpr int NW = THREADS / 32;
  constexpr int LOG2T = (T == 512) ? 9 : (T == 1024) ? 10 : (T == 2048) ? 11 : (T == 4096) ? 12
                      : (T == 8192) ? 13 : (T == 16384) ? 14 : 15;
  static_assert((1 << LOG2T) == T, "T must be a power of two");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* tvals = reinterpret_cast<V*>(smem_raw);                                // T values
  int32_t* tkeys = reinterpret_cast<int32_t*>(smem_raw + sizeof(V) * T);    // T keys
  uint64_t* sortbuf = reinterpret_cast<uint64_t*>(tkeys);                   // aliases keys (<= T/2 entries)
  using BlockScan = cub::BlockScan<int, THREADS>;
  __shared__ typename BlockScan::TempStorage scan_tmp;
  __shared__ int s_total;

  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t r = blockIdx.x; r < nrows_bin; r += gridDim.x) {
    const int64_t i = rows[r];
    for (int e = threadIdx.x; e < T; e += THREADS) {
      tkeys[e] = kEmptyKey;
      tvals[e] = SR::zero();
    }
    __syncthreads();
    const int64_t se = src.seg_end(i);
    for (int64_t s = src.seg_begin(i) + wid; s < se; s += NW) {
      int64_t b, len;
      const int32_t* cols;
      const V* vals;
      V mult;
      src.segment(i, s, b, len, cols, vals, mult);
      for (int64_t u = b + lane; u < b + len; u += 32) {
        const int32_t c = __ldg(cols + u);
        const V v = src.item(mult, vals[u]);
        uint32_t h = hash_slot((uint32_t)c, LOG2T);
        for (;;) {
          const int32_t k = *reinterpret_cast<volatile int32_t*>(&tkeys[h]);
          if (k == c) break;
          if (k == kEmptyKey) {
            const int32_t prev = atomicCAS(&tkeys[h], kEmptyKey, c);
            if (prev == kEmptyKey || prev == c) break;
          }
          h = (h + 1) & (T - 1);
        }
        atomic_accumulate<SR, true>(&tvals[h], v);
      }
    }
    __syncthreads();
    // compaction: gather occupied non-zero slots
    int my_slots[SPT];
    int cnt = 0;
#pragma unroll
    for (int q = 0; q < SPT; ++q) {
      const int e = threadIdx.x * SPT + q;
      const int32_t k = tkeys[e];
      my_slots[q] = -1;
      if (k != kEmptyKey && !SR::is_zero(tvals[e])) {
        my_slots[q] = e;
        ++cnt;
      }
    }
    int first, total;
    BlockScan(scan_tmp).ExclusiveSum(cnt, first, total);
    uint32_t my_keys[SPT];
#pragma unroll
    for (int q = 0; q < SPT; ++q) my_keys[q] = my_slots[q] >= 0 ? (uint32_t)tkeys[my_slots[q]] : 0u;
    __syncthreads();  // all keys read before the sort buffer overwrites them
    int w = first;
#pragma unroll
    for (int q = 0; q < SPT; ++q) {
      if (my_slots[q] >= 0) {
        sortbuf[w++] = ((uint64_t)my_keys[q] << 32) | (uint32_t)my_slots[q];
      }
    }
    if (threadIdx.x == 0) s_total = total;
    __syncthreads();
    const int n = s_total;
    block_bitonic_sort<THREADS>(sortbuf, n);
    const int64_t o = off[i];
    for (int e = threadIdx.x; e < n; e += THREADS) {
      const uint64_t kk = sortbuf[e];
      out_cols[o + e] = (int32_t)(kk >> 32);
      out_vals[o + e] = tvals[(uint32_t)kk];
    }
    if (threadIdx.x == 0) rownnz[i] = n;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K5 bin 6: dense accumulator in global memory.  Each CTA owns a slab of
// ncols values + an ncols-bit presence bitmap (zeroed by the host, restored
// to zero/zero() after each row so the slab is reusable).
// ---------------------------------------------------------------------------
template <class SR, class Src, int THREADS>
__global__ void __launch_bounds__(THREADS) dense_rows_kernel(Src src, const int64_t* __restrict__ rows,
                                                             int64_t nrows_bin, int64_t ncols,
                                                             typename SR::value_type* __restrict__ slabs,
                                                             uint32_t* __restrict__ bitmaps,
                                                             const int64_t* __restrict__ off,
                                                             int32_t* __restrict__ out_cols,
                                                             typename SR::value_type* __restrict__ out_vals,
                                                             int64_t* __restrict__ rownnz) {
  using V = typename SR::value_type;
  constexpr int NW = THREADS / 32;
  using BlockScan = cub::BlockScan<int, THREADS>;
  __shared__ typename BlockScan::TempStorage scan_tmp;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t nwords = (ncols + 31) >> 5;
  V* dv = slabs + (int64_t)blockIdx.x * ncols;
  uint32_t* bm = bitmaps + (int64_t)blockIdx.x * nwords;
  for (int64_t e = threadIdx.x; e < ncols; e += THREADS) dv[e] = SR::zero();
  __syncthreads();
  for (int64_t r = blockIdx.x; r < nrows_bin; r += gridDim.x) {
    const int64_t i = rows[r];
    const int64_t se = src.seg_end(i);
    for (int64_t s = src.seg_begin(i) + wid; s < se; s += NW) {
      int64_t b, len;
      const int32_t* cols;
      const V* vals;
      V mult;
      src.segment(i, s, b, len, cols, vals, mult);
      for (int64_t u = b + lane; u < b + len; u += 32) {
        const int32_t c = __ldg(cols + u);
        const V v = src.item(mult, vals[u]);
        atomic_accumulate<SR, false>(&dv[c], v);
        atomicOr(&bm[c >> 5], 1u << (c & 31));
      }
    }
    __syncthreads();
    const int64_t o = off[i];
    int64_t written = 0;
    for (int64_t w0 = 0; w0 < nwords; w0 += THREADS) {
      const int64_t w = w0 + threadIdx.x;
      uint32_t bits = w < nwords ? bm[w] : 0u;
      uint32_t keep = 0;
      for (uint32_t x = bits; x; x &= x - 1) {
        const int bit = __ffs(x) - 1;
        if (!SR::is_zero(dv[(w << 5) + bit])) keep |= 1u << bit;
      }
      const int cnt = __popc(keep);
      int first, total;
      BlockScan(scan_tmp).ExclusiveSum(cnt, first, total);
      int64_t p = o + written + first;
      for (uint32_t x = bits; x; x &= x - 1) {
        const int bit = __ffs(x) - 1;
        const int64_t c = (w << 5) + bit;
        if (keep & (1u << bit)) {
          out_cols[p] = (int32_t)c;
          out_vals[p] = dv[c];
          ++p;
        }
        dv[c] = SR::zero();
      }
      if (bits) bm[w] = 0u;
      written += total;
      __syncthreads();
    }
    if (threadIdx.x == 0) rownnz[i] = written;
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K7: compaction scratch -> exact CSR (warp per row, 16-byte stores when the
// run is long enough)
// ---------------------------------------------------------------------------
template <class V>
__global__ void __launch_bounds__(256) compact_rows_kernel(int64_t nrows, const int64_t* __restrict__ off,
                                                           const int64_t* __restrict__ rowptr,
                                                           const int32_t* __restrict__ sc_cols,
                                                           const V* __restrict__ sc_vals,
                                                           int32_t* __restrict__ cols, V* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nrows; i += nwarps) {
    const int64_t d = rowptr[i];
    const int64_t n = rowptr[i + 1] - d;
    const int64_t s = off[i];
    for (int64_t e = lane; e < n; e += 32) {
      cols[d + e] = sc_cols[s + e];
      vals[d + e] = sc_vals[s + e];
    }
  }
}

}  // namespace spg
