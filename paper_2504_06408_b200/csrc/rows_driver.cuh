// Host driver for the row-accumulation pipeline in accumulate.cuh: runs
// analyse -> bin -> numeric (row-batched under a scratch budget) -> compact
// for any Source, producing an exact-size device CSR.
#pragma once
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <vector>

#include "accumulate.cuh"

namespace spg {

struct PhaseTimer {
  spg_ctx* c;
  bool on;
  explicit PhaseTimer(spg_ctx* ctx, bool enabled) : c(ctx), on(enabled) {
    if (on)
      for (int k = 0; k < 4; ++k)
        if (!c->ev[k]) SPG_CUDA(cudaEventCreate(&c->ev[k]));
  }
  void mark(int k) {
    if (on) SPG_CUDA(cudaEventRecord(c->ev[k], c->stream));
  }
  float between(int a, int b) {
    if (!on) return 0.f;
    SPG_CUDA(cudaEventSynchronize(c->ev[b]));
    float ms = 0.f;
    SPG_CUDA(cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]));
    return ms;
  }
};

template <class T>
inline void exclusive_scan(spg_ctx* c, const T* in, T* out, int64_t n) {
  size_t bytes = 0;
  SPG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, c->stream));
  ensure_cub_tmp(c, bytes);
  SPG_CUDA(cub::DeviceScan::ExclusiveSum(c->cub_tmp, bytes, in, out, n, c->stream));
  ++c->launches;
}

inline int grid_for(spg_ctx* c, int64_t work_items, int per_block, int max_waves = 16) {
  const int64_t want = (work_items + per_block - 1) / per_block;
  const int64_t cap = (int64_t)c->sm_count * max_waves;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, cap));
}

template <class SR, class Src, int T, int THREADS>
void launch_hash(spg_ctx* c, const Src& src, const int64_t* rows, int64_t n, const int64_t* off,
                 int32_t* sc_cols, typename SR::value_type* sc_vals, int64_t* rownnz) {
  using V = typename SR::value_type;
  const size_t smem = (size_t)T * (sizeof(V) + sizeof(int32_t));
  auto kern = hash_rows_kernel<SR, Src, T, THREADS>;
  static bool configured = false;  // per template instantiation
  if (!configured) {
    SPG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = true;
  }
  int per_sm = 1;
  SPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, THREADS, smem));
  const int64_t cap = (int64_t)c->sm_count * std::max(per_sm, 1);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(n, cap));
  kern<<<grid, THREADS, smem, c->stream>>>(src, rows, n, off, sc_cols, sc_vals, rownnz);
  SPG_LAUNCH_CHECK();
  ++c->launches;
}

// Runs the pipeline for rows [0, src.nrows) with output width ncols_out.
template <class SR, class Src>
void run_rows(spg_ctx* c, const Src& src, int64_t ncols_out, spg_dcsr* out, spg_mult_stats* st) {
  using V = typename SR::value_type;
  const int64_t m = src.nrows;
  PhaseTimer tm(c, st != nullptr);
  const uint64_t launches0 = c->launches;
  tm.mark(0);

  out->nrows = m;
  out->ncols = ncols_out;
  out->nnz = 0;
  out->ptr = dalloc<int64_t>(c, m + 1);
  out->idx = nullptr;
  out->vals = nullptr;
  if (m == 0) {
    SPG_CUDA(cudaMemsetAsync(out->ptr, 0, sizeof(int64_t), c->stream));
    out->idx = dalloc<int32_t>(c, 1);
    out->vals = dalloc<V>(c, 1);
    if (st) *st = spg_mult_stats{};
    return;
  }

  // K1 analyse
  DBuf<int64_t> prods(c, m), ub(c, m + 1), off(c, m + 1), rownnz(c, m + 1);
  DBuf<uint8_t> bins(c, m);
  {
    const int grid = grid_for(c, m, 8);
    analyse_rows_kernel<SR, Src><<<grid, 256, 0, c->stream>>>(src, ncols_out, prods.p, ub.p, bins.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
  }
  SPG_CUDA(cudaMemsetAsync(ub.p + m, 0, sizeof(int64_t), c->stream));
  SPG_CUDA(cudaMemsetAsync(rownnz.p + m, 0, sizeof(int64_t), c->stream));
  exclusive_scan(c, ub.p, off.p, m + 1);  // off[m] = total scratch entries
  // products total (for stats) via scan on prods is not needed on the hot
  // path; F is reduced from the same array into a scalar below.
  DBuf<unsigned long long> counts(c, 2 * kNumBins);
  SPG_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(unsigned long long) * 2 * kNumBins, c->stream));
  {
    const int grid = grid_for(c, m, 1024, 2);
    bin_count_kernel<<<grid, 1024, 0, c->stream>>>(bins.p, m, counts.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
  }
  unsigned long long hcounts[kNumBins];
  int64_t scratch_total = 0;
  SPG_CUDA(cudaMemcpyAsync(hcounts, counts.p, sizeof(hcounts), cudaMemcpyDeviceToHost, c->stream));
  SPG_CUDA(cudaMemcpyAsync(&scratch_total, off.p + m, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  SPG_CUDA(cudaStreamSynchronize(c->stream));
  int64_t products = 0;
  if (st) {
    size_t bytes = 0;
    DBuf<int64_t> fsum(c, 1);
    SPG_CUDA(cub::DeviceReduce::Sum(nullptr, bytes, prods.p, fsum.p, m, c->stream));
    ensure_cub_tmp(c, bytes);
    SPG_CUDA(cub::DeviceReduce::Sum(c->cub_tmp, bytes, prods.p, fsum.p, m, c->stream));
    ++c->launches;
    products = d2h_scalar(c, fsum.p);
  }

  // Row batches under the scratch budget (contiguous row ranges).
  size_t budget = c->scratch_budget;
  if (budget == 0) {
    size_t fr = 0, tot = 0;
    SPG_CUDA(cudaMemGetInfo(&fr, &tot));
    budget = (size_t)(fr * 0.4);
  }
  const size_t per_entry = sizeof(int32_t) + sizeof(V);
  std::vector<int64_t> cuts{0};
  if ((size_t)scratch_total * per_entry <= budget) {
    cuts.push_back(m);
  } else {
    std::vector<int64_t> hoff(m + 1);
    SPG_CUDA(cudaMemcpyAsync(hoff.data(), off.p, sizeof(int64_t) * (m + 1), cudaMemcpyDeviceToHost, c->stream));
    SPG_CUDA(cudaStreamSynchronize(c->stream));
    const int64_t cap_entries = std::max<int64_t>(1, (int64_t)(budget / per_entry));
    int64_t r0 = 0;
    while (r0 < m) {
      // largest r1 with hoff[r1] - hoff[r0] <= cap (at least one row)
      int64_t r1 = std::upper_bound(hoff.begin() + r0 + 1, hoff.end(), hoff[r0] + cap_entries) - hoff.begin() - 1;
      if (r1 <= r0) r1 = r0 + 1;
      cuts.push_back(r1);
      r0 = r1;
    }
  }
  const bool batched = cuts.size() > 2;
  tm.mark(1);

  // Dense slabs (bin 6), sized once for all batches.
  const int64_t n6_total = (int64_t)hcounts[6];
  int dense_grid = 0;
  DBuf<V> slabs;
  DBuf<uint32_t> bitmaps;
  const int64_t nwords = (ncols_out + 31) / 32;
  if (n6_total > 0) {
    const size_t per_cta = (size_t)ncols_out * sizeof(V) + (size_t)nwords * 4;
    const size_t slab_budget = (size_t)4 << 30;
    dense_grid = (int)std::max<int64_t>(1, std::min<int64_t>({n6_total, (int64_t)c->sm_count * 2,
                                                             (int64_t)(slab_budget / std::max<size_t>(per_cta, 1))}));
    slabs = DBuf<V>(c, (size_t)dense_grid * ncols_out);
    bitmaps = DBuf<uint32_t>(c, (size_t)dense_grid * nwords);
    SPG_CUDA(cudaMemsetAsync(bitmaps.p, 0, sizeof(uint32_t) * dense_grid * nwords, c->stream));
  }

  DBuf<int64_t> lists(c, m);
  DBuf<unsigned long long> cursor(c, kNumBins);
  std::vector<DBuf<int32_t>> part_cols;
  std::vector<DBuf<V>> part_vals;
  std::vector<int64_t> part_nnz;
  float ms_numeric = 0.f, ms_compact = 0.f;

  for (size_t bi = 0; bi + 1 < cuts.size(); ++bi) {
    const int64_t r0 = cuts[bi], r1 = cuts[bi + 1];
    int64_t bcount[kNumBins];
    if (!batched) {
      for (int b = 0; b < kNumBins; ++b) bcount[b] = (int64_t)hcounts[b];
    } else {
      SPG_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(unsigned long long) * kNumBins, c->stream));
      bin_count_kernel<<<grid_for(c, r1 - r0, 1024, 2), 1024, 0, c->stream>>>(bins.p + r0, r1 - r0, counts.p);
      SPG_LAUNCH_CHECK();
      ++c->launches;
      unsigned long long hc[kNumBins];
      SPG_CUDA(cudaMemcpyAsync(hc, counts.p, sizeof(hc), cudaMemcpyDeviceToHost, c->stream));
      SPG_CUDA(cudaStreamSynchronize(c->stream));
      for (int b = 0; b < kNumBins; ++b) bcount[b] = (int64_t)hc[b];
    }
    unsigned long long base[kNumBins];
    unsigned long long acc = 0;
    for (int b = 0; b < kNumBins; ++b) {
      base[b] = acc;
      if (b > 0) acc += bcount[b];
    }
    SPG_CUDA(cudaMemcpyAsync(cursor.p, base, sizeof(base), cudaMemcpyHostToDevice, c->stream));
    // lists hold absolute row ids; bins.p + r0 scanning yields ids relative to r0
    bin_scatter_kernel<<<grid_for(c, r1 - r0, 1024, 2), 1024, 0, c->stream>>>(bins.p + r0, r1 - r0,
                                                                             cursor.p, lists.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;

    // scratch for this batch; offsets are relative to off[r0]
    int64_t sc_lo = 0, sc_hi = scratch_total;
    if (batched) {
      SPG_CUDA(cudaMemcpyAsync(&sc_lo, off.p + r0, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
      SPG_CUDA(cudaMemcpyAsync(&sc_hi, off.p + r1, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
      SPG_CUDA(cudaStreamSynchronize(c->stream));
    }
    DBuf<int32_t> sc_cols(c, (size_t)(sc_hi - sc_lo));
    DBuf<V> sc_vals(c, (size_t)(sc_hi - sc_lo));
    // Kernels index scratch with the global offsets off[i]; shift the base
    // pointers so this batch's window [sc_lo, sc_hi) is what they address.
    int32_t* sccb = sc_cols.p - sc_lo;
    V* scvb = sc_vals.p - sc_lo;
    // Row ids in `lists` are relative to r0 (bin_scatter ran over bins + r0):
    // hand the kernels views that start at row r0.
    Src bsrc = src;
    rebase_source(bsrc, r0);
    const int64_t* offb = off.p + r0;
    int64_t* nnzb = rownnz.p + r0;

    const int64_t* lb = lists.p;
    if (bcount[1] > 0) {
      esc_warp_kernel<SR, Src><<<grid_for(c, bcount[1], 8), 256, 0, c->stream>>>(
          bsrc, lb + base[1], bcount[1], offb, sccb, scvb, nnzb);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    if (bcount[2] > 0) launch_hash<SR, Src, bin_table<V>(2), 128>(c, bsrc, lb + base[2], bcount[2], offb, sccb, scvb, nnzb);
    if (bcount[3] > 0) launch_hash<SR, Src, bin_table<V>(3), 256>(c, bsrc, lb + base[3], bcount[3], offb, sccb, scvb, nnzb);
    if (bcount[4] > 0) launch_hash<SR, Src, bin_table<V>(4), 512>(c, bsrc, lb + base[4], bcount[4], offb, sccb, scvb, nnzb);
    if (bcount[5] > 0) launch_hash<SR, Src, bin_table<V>(5), 1024>(c, bsrc, lb + base[5], bcount[5], offb, sccb, scvb, nnzb);
    if (bcount[6] > 0) {
      const int g = (int)std::min<int64_t>(dense_grid, bcount[6]);
      dense_rows_kernel<SR, Src, 1024><<<g, 1024, 0, c->stream>>>(bsrc, lb + base[6], bcount[6], ncols_out,
                                                                 slabs.p, bitmaps.p, offb, sccb, scvb, nnzb);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    // rows of bin 0 are never visited by a numeric kernel: nnz 0
    if (bcount[0] > 0) {
      zero_empty_rows_kernel<<<grid_for(c, r1 - r0, 256, 4), 256, 0, c->stream>>>(bins.p + r0, r1 - r0, nnzb);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    tm.mark(2);
    ms_numeric += tm.between(1, 2);

    if (!batched) {
      exclusive_scan(c, rownnz.p, out->ptr, m + 1);
      int64_t nnz = d2h_scalar(c, out->ptr + m);
      out->nnz = nnz;
      out->idx = dalloc<int32_t>(c, (size_t)nnz);
      out->vals = dalloc<V>(c, (size_t)nnz);
      compact_rows_kernel<V><<<grid_for(c, m, 8), 256, 0, c->stream>>>(
          m, off.p, out->ptr, sccb, scvb, out->idx, static_cast<V*>(out->vals));
      SPG_LAUNCH_CHECK();
      ++c->launches;
    } else {
      // compact this batch into an exact buffer; the exclusive scan over
      // rownnz[r0 .. r1] ends with the batch total (the last input, which
      // belongs to the next batch, is excluded by construction)
      DBuf<int64_t> bptr(c, r1 - r0 + 1);
      exclusive_scan(c, rownnz.p + r0, bptr.p, r1 - r0 + 1);
      const int64_t bn = d2h_scalar(c, bptr.p + (r1 - r0));
      DBuf<int32_t> pc(c, (size_t)bn);
      DBuf<V> pv(c, (size_t)bn);
      compact_rows_kernel<V><<<grid_for(c, r1 - r0, 8), 256, 0, c->stream>>>(
          r1 - r0, offb, bptr.p, sccb, scvb, pc.p, pv.p);
      SPG_LAUNCH_CHECK();
      ++c->launches;
      part_cols.push_back(std::move(pc));
      part_vals.push_back(std::move(pv));
      part_nnz.push_back(bn);
    }
    tm.mark(3);
    ms_compact += tm.between(2, 3);
    tm.mark(1);
  }

  if (batched) {
    exclusive_scan(c, rownnz.p, out->ptr, m + 1);
    const int64_t nnz = d2h_scalar(c, out->ptr + m);
    out->nnz = nnz;
    out->idx = dalloc<int32_t>(c, (size_t)nnz);
    out->vals = dalloc<V>(c, (size_t)nnz);
    int64_t pos = 0;
    for (size_t k = 0; k < part_nnz.size(); ++k) {
      if (part_nnz[k] == 0) continue;
      SPG_CUDA(cudaMemcpyAsync(out->idx + pos, part_cols[k].p, sizeof(int32_t) * part_nnz[k],
                               cudaMemcpyDeviceToDevice, c->stream));
      SPG_CUDA(cudaMemcpyAsync(static_cast<V*>(out->vals) + pos, part_vals[k].p, sizeof(V) * part_nnz[k],
                               cudaMemcpyDeviceToDevice, c->stream));
      pos += part_nnz[k];
    }
    tm.mark(3);
    ms_compact += tm.between(1, 3);
  }
  if (st) {
    tm.mark(3);
    st->products = products;
    st->nnz_out = out->nnz;
    for (int b = 0; b < 8; ++b) st->rows_per_bin[b] = b < kNumBins ? (int64_t)hcounts[b] : 0;
    st->ms_numeric = ms_numeric;
    st->ms_compact = ms_compact;
    st->ms_total = tm.between(0, 3);
    st->ms_analyse = st->ms_total - ms_numeric - ms_compact;
    st->kernels = (int64_t)(c->launches - launches0);
  }
}

}  // namespace spg
