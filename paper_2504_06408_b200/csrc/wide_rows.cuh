// Sort-based fallback for rows that no shared-memory accumulator holds: an
// output width too large for dense column panels (the per-segment panel
// offsets no longer fit next to a panel) AND more distinct columns than the
// largest hash table (e.g. ER max-times at 1x1: 4 M columns, 16-byte values,
// the Poisson tail of rows with > 4096 outputs).
//
// The rows' products are expanded into HBM as (list row, column) keys in
// generation order — A's row order, then B's — so one stable device radix
// sort groups equal keys in the reference's fold order
// (local_spgemm.hpp:107-155); each run folds left to right with SR::add,
// results equal to SR::is_zero are dropped, and every row then claims its
// exact nnz from the RowOut like any other bin (U slot, exact claim, or
// straight into C on the second pass).  Rows are processed in batches whose
// products fit a fixed HBM budget.
#pragma once
#include <cub/cub.cuh>

#include "accumulate.cuh"

namespace spg {

// warp per list row: products of row rows[j] at poffs[j] .. poffs[j + 1]
template <class SR, class Src>
__global__ void __launch_bounds__(256) wide_expand_kernel(Src src, const int64_t* __restrict__ rows, int64_t nr,
                                                          const int64_t* __restrict__ poffs,
                                                          uint64_t* __restrict__ keys,
                                                          typename SR::value_type* __restrict__ vals) {
  using V = typename SR::value_type;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = warp; j < nr; j += nwarps) {
    const int64_t i = rows[j];
    int64_t o = poffs[j];
    const uint64_t hi = (uint64_t)j << 32;
    for (int64_t s = src.seg_begin(i), se = src.seg_end(i); s < se; ++s) {
      int64_t b;
      int len, sid;
      V mult;
      src.seg(i, s, -1, b, len, sid, mult);
      for (int t = lane; t < len; t += 32) {
        SPG_DCHECK(o + t < poffs[j + 1]);  // the row's products fit its counted range
        keys[o + t] = hi | (uint32_t)src.col(sid, b + t);
        vals[o + t] = src.item(mult, src.val(sid, b + t));
      }
      o += len;
    }
  }
}

static __global__ void wide_heads_kernel(int64_t n, const uint64_t* __restrict__ k, int64_t* __restrict__ f) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    f[p] = p == 0 || k[p] != k[p - 1];
}

// run u = sorted positions [head(u), head(u + 1)): fold, keep flag, key
template <class SR>
__global__ void __launch_bounds__(256) wide_fold_kernel(int64_t n, const int64_t* __restrict__ f,
                                                        const int64_t* __restrict__ pos,
                                                        const uint64_t* __restrict__ skeys,
                                                        const uint32_t* __restrict__ order,
                                                        const typename SR::value_type* __restrict__ vin,
                                                        uint64_t* __restrict__ ukeys,
                                                        typename SR::value_type* __restrict__ uvals,
                                                        int64_t* __restrict__ keep) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    if (!f[p]) continue;
    const uint64_t key = skeys[p];
    typename SR::value_type acc = vin[order[p]];
    for (int64_t q = p + 1; q < n && skeys[q] == key; ++q) acc = SR::add(acc, vin[order[q]]);
    const int64_t u = pos[p];
    ukeys[u] = key;
    uvals[u] = acc;
    keep[u] = !SR::is_zero(acc);
  }
}

// per list row: kept entries [kb[j], kb[j + 1]) of the kept order; claims them
template <class V>
__global__ void wide_claim_kernel(int64_t nr, const int64_t* __restrict__ rows, const int64_t* __restrict__ poffs,
                                  const int64_t* __restrict__ pos, const int64_t* __restrict__ kpos, int64_t n,
                                  int64_t nu, int64_t nkept, int64_t* __restrict__ kb, int64_t* __restrict__ base,
                                  RowOut<V> o) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nr; j += (int64_t)gridDim.x * blockDim.x) {
    auto kept_at = [&](int64_t prod) {  // kept entries before the first run at sorted position prod
      if (prod >= n) return nkept;
      const int64_t u = pos[prod];
      return u >= nu ? nkept : kpos[u];
    };
    const int64_t b = kept_at(poffs[j]), e = kept_at(poffs[j + 1]);
    kb[j] = b;
    const int64_t cnt = e - b;
    const int64_t i = rows[j];
    o.rownnz[i] = cnt;
    base[j] = o.writes() ? o.claim_row(i, cnt) : -1;
  }
}

template <class V>
__global__ void wide_store_kernel(int64_t nu, const int64_t* __restrict__ keep, const int64_t* __restrict__ kpos,
                                  const uint64_t* __restrict__ ukeys, const V* __restrict__ uvals,
                                  const int64_t* __restrict__ kb, const int64_t* __restrict__ base, RowOut<V> o) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nu; u += (int64_t)gridDim.x * blockDim.x) {
    if (!keep[u]) continue;
    const int64_t j = (int64_t)(ukeys[u] >> 32);
    if (base[j] < 0) continue;
    SPG_DCHECK(kpos[u] >= kb[j]);
    const int64_t d = base[j] + (kpos[u] - kb[j]);
    o.cols[d] = (int32_t)(uint32_t)ukeys[u];
    o.vals[d] = uvals[u];
  }
}

static __global__ void relabel_bin_kernel(uint8_t* __restrict__ bins, int64_t n, uint8_t from, uint8_t to) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (bins[i] == from) bins[i] = to;
}

static __global__ void wide_gather_kernel(const int64_t* __restrict__ rows, int64_t n, const int64_t* __restrict__ prods,
                                   int64_t* __restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    out[j] = prods[rows[j]];
}

static __global__ void wide_iota_kernel(uint32_t* __restrict__ a, int64_t n) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    a[p] = (uint32_t)p;
}

// rows[0 .. n) (device list), prods = per-row product counts (indexed by row
// id); runs on the context stream.
template <class SR, class Src>
void run_wide_rows(spg_ctx* c, const Src& src, const int64_t* rows, int64_t n, const int64_t* prods,
                   const RowOut<typename SR::value_type>& o) {
  using V = typename SR::value_type;
  if (n <= 0) return;
  NvtxRange nv("spg:wide rows (sort fallback)");
  cudaStream_t s = c->stream;
  auto grid = [&](int64_t items) {
    return (int)std::max<int64_t>(1, std::min<int64_t>((items + 255) / 256, (int64_t)c->sm_count * 8));
  };
  std::vector<int64_t> hf((size_t)n);
  {
    DBuf<int64_t> g(c, n);
    wide_gather_kernel<<<grid(n), 256, 0, s>>>(rows, n, prods, g.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
    SPG_CUDA(cudaMemcpyAsync(hf.data(), g.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, s));
    SPG_CUDA(cudaStreamSynchronize(s));
  }
  constexpr size_t kPerProduct = 8 + 8 + 4 + 4 + sizeof(V) + 8 + 8 + 8 + 8 + sizeof(V) + 8;
  const int64_t budget = std::max<int64_t>(int64_t(1) << 20, std::min<int64_t>(int64_t(1) << 28,
                                           (int64_t)(mem_available(c) * 0.15 / kPerProduct)));
  for (int64_t j0 = 0; j0 < n;) {
    int64_t j1 = j0, T = 0;
    while (j1 < n && (j1 == j0 || T + hf[(size_t)j1] <= budget)) T += hf[(size_t)j1++];
    if (T >= (int64_t(1) << 31)) fail(SPG_ERR_OOM, "wide row: more than 2^31 products in one row");
    const int64_t nr = j1 - j0;
    std::vector<int64_t> hp((size_t)nr + 1, 0);
    for (int64_t j = 0; j < nr; ++j) hp[(size_t)j + 1] = hp[(size_t)j] + hf[(size_t)(j0 + j)];
    DBuf<int64_t> poffs(c, nr + 1);
    SPG_CUDA(cudaMemcpyAsync(poffs.p, hp.data(), sizeof(int64_t) * (nr + 1), cudaMemcpyHostToDevice, s));
    DBuf<uint64_t> keys(c, T), skeys(c, T);
    DBuf<uint32_t> order(c, T), sorder(c, T);
    DBuf<V> vals(c, T);
    const int64_t* lrows = rows + j0;
    wide_expand_kernel<SR, Src><<<(int)std::min<int64_t>((nr + 7) / 8, (int64_t)c->sm_count * 16), 256, 0, s>>>(
        src, lrows, nr, poffs.p, keys.p, vals.p);
    SPG_LAUNCH_CHECK();
    wide_iota_kernel<<<grid(T), 256, 0, s>>>(order.p, T);
    SPG_LAUNCH_CHECK();
    int end_bit = 32;
    while ((int64_t{1} << (end_bit - 32)) < nr) ++end_bit;
    size_t bytes = 0;
    SPG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, skeys.p, order.p, sorder.p, (int)T, 0, end_bit,
                                             s));
    ensure_cub_tmp(c, bytes);
    SPG_CUDA(cub::DeviceRadixSort::SortPairs(c->cub_tmp, bytes, keys.p, skeys.p, order.p, sorder.p, (int)T, 0,
                                             end_bit, s));
    keys.reset();
    order.reset();
    DBuf<int64_t> f(c, T), pos(c, T);
    wide_heads_kernel<<<grid(T), 256, 0, s>>>(T, skeys.p, f.p);
    SPG_LAUNCH_CHECK();
    exclusive_scan(c, f.p, pos.p, T);
    const int64_t nu = d2h_scalar(c, pos.p + T - 1) + d2h_scalar(c, f.p + T - 1);
    DBuf<uint64_t> ukeys(c, nu);
    DBuf<V> uvals(c, nu);
    DBuf<int64_t> keep(c, nu), kpos(c, nu);
    wide_fold_kernel<SR><<<grid(T), 256, 0, s>>>(T, f.p, pos.p, skeys.p, sorder.p, vals.p, ukeys.p, uvals.p, keep.p);
    SPG_LAUNCH_CHECK();
    exclusive_scan(c, keep.p, kpos.p, nu);
    const int64_t nkept = d2h_scalar(c, kpos.p + nu - 1) + d2h_scalar(c, keep.p + nu - 1);
    DBuf<int64_t> kb(c, nr), base(c, nr);
    wide_claim_kernel<V><<<grid(nr), 256, 0, s>>>(nr, lrows, poffs.p, pos.p, kpos.p, T, nu, nkept, kb.p, base.p, o);
    SPG_LAUNCH_CHECK();
    if (o.cols != nullptr) {  // (RowOut::writes() is device-only: its host stub would exit)
      wide_store_kernel<V><<<grid(nu), 256, 0, s>>>(nu, keep.p, kpos.p, ukeys.p, uvals.p, kb.p, base.p, o);
      SPG_LAUNCH_CHECK();
    }
    c->launches += 7;
    j0 = j1;
  }
}

}  // namespace spg
