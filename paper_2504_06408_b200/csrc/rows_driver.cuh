// Host driver for the row-accumulation pipeline in accumulate.cuh: runs
// analyse -> bin -> numeric (bins on concurrent streams) -> compact for any
// Source, producing an exact CSR; falls back to an exact two-pass (count,
// then write into C) mode when the scratch would exceed the budget.
#pragma once
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "accumulate.cuh"
#include "bitmap_rank.cuh"

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

}  // namespace spg
#include "wide_rows.cuh"  // uses exclusive_scan above
namespace spg {

// Forked side streams so independent bins overlap on the SMs.
struct StreamFork {
  spg_ctx* c;
  int n;
  StreamFork(spg_ctx* ctx, int count) : c(ctx), n(count) {
    for (int k = 0; k < n; ++k) {
      if (!c->aux[k]) SPG_CUDA(cudaStreamCreateWithFlags(&c->aux[k], cudaStreamNonBlocking));
      if (!c->aux_ev[k]) SPG_CUDA(cudaEventCreateWithFlags(&c->aux_ev[k], cudaEventDisableTiming));
    }
    if (!c->fork_ev) SPG_CUDA(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
    SPG_CUDA(cudaEventRecord(c->fork_ev, c->stream));
    for (int k = 0; k < n; ++k) SPG_CUDA(cudaStreamWaitEvent(c->aux[k], c->fork_ev, 0));
  }
  cudaStream_t operator[](int k) const { return c->aux[k % n]; }
  void join() {
    for (int k = 0; k < n; ++k) {
      SPG_CUDA(cudaEventRecord(c->aux_ev[k], c->aux[k]));
      SPG_CUDA(cudaStreamWaitEvent(c->stream, c->aux_ev[k], 0));
    }
  }
};

template <class K>
inline void set_smem(K kern, size_t smem) {
  // static + dynamic above 48 KB needs the opt-in (set unconditionally: cheap, idempotent)
  if (smem > 16 * 1024) SPG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
}

template <class K>
inline int resident_grid(spg_ctx* c, K kern, int threads, size_t smem, int64_t work) {
  int per_sm = 1;
  SPG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem));
  const int64_t cap = (int64_t)c->sm_count * std::max(per_sm, 1);
  return (int)std::max<int64_t>(1, std::min<int64_t>(work, cap));
}

// gtab (optional, gtab_slots entries, zero and left zero): per-CTA value
// tables in global memory for semirings with a native L2 reduction
// (has_red_global: fp64 +); the shared-memory table is used otherwise, or
// when the resident grid needs more slots than gtab holds.
template <class SR, class Src, int T, int THREADS, bool OPT = false>
void launch_hash(spg_ctx* c, cudaStream_t s, const Src& src, const int64_t* rows, int64_t n, int cap, int end_bit,
                 const RowOut<typename SR::value_type>& out, unsigned long long* ovf_n = nullptr,
                 int64_t* ovf_rows = nullptr, typename SR::value_type* gtab = nullptr, size_t gtab_slots = 0) {
  using V = typename SR::value_type;
  const size_t fixed = (size_t)T * (sizeof(V) + sizeof(int32_t) + sizeof(uint32_t)) +
                       ((sizeof(typename HashSort<T, THREADS>::Tmp) + 15) & ~size_t(15)) + 64;
  const size_t per = SegCache<SR, Src>::bytes_per_seg(1);
  const size_t limit = 220 * 1024;
  const int fit = fixed < limit ? (int)((limit - fixed) / per) : 0;
  cap = std::min(cap, fit) & ~3;
  if (cap < 32) fail(SPG_ERR_INTERNAL, "hash bin: no shared memory left for the segment cache");
  const size_t smem = fixed + (size_t)cap * per;
  if constexpr (has_red_global<SR>::value) {
    static const int gred_on = [] {  // SPG_HASH_GRED=1: L2-reduction tables (config 4: 231 vs 222 ms, kept off)
      const char* e = std::getenv("SPG_HASH_GRED");
      return e ? std::atoi(e) : 0;
    }();
    if (gred_on && gtab) {
      auto kern = hash_rows_kernel<SR, Src, T, THREADS, OPT, true>;
      set_smem(kern, smem);
      const int grid = resident_grid(c, kern, THREADS, smem, n);
      if ((size_t)grid * T <= gtab_slots) {
        kern<<<grid, THREADS, smem, s>>>(src, rows, n, cap, end_bit, out, ovf_n, ovf_rows, gtab);
        SPG_LAUNCH_CHECK();
        ++c->launches;
        return;
      }
    }
  }
  auto kern = hash_rows_kernel<SR, Src, T, THREADS, OPT, false>;
  set_smem(kern, smem);
  kern<<<resident_grid(c, kern, THREADS, smem, n), THREADS, smem, s>>>(src, rows, n, cap, end_bit, out, ovf_n,
                                                                        ovf_rows, nullptr);
  SPG_LAUNCH_CHECK();
  ++c->launches;
}

template <class SR, class Src, int THREADS, int ITEMS>
void launch_esc(spg_ctx* c, cudaStream_t s, const Src& src, const int64_t* rows, int64_t n, int end_bit,
                const RowOut<typename SR::value_type>& out) {
  const size_t smem = sizeof(EscSmem<SR, THREADS, ITEMS>);
  auto kern = esc_block_kernel<SR, Src, THREADS, ITEMS>;
  set_smem(kern, smem);
  kern<<<resident_grid(c, kern, THREADS, smem, n), THREADS, smem, s>>>(src, rows, n, end_bit, out);
  SPG_LAUNCH_CHECK();
  ++c->launches;
}

// Dense-panel geometry: (panel width, CTA size, smem budget per CTA).
// cfg 0: 128 KB panel, 1024 threads, 1 CTA/SM; cfg 1: 64 KB, 512 threads,
// 2 CTAs/SM; cfg 2: 32 KB, 512 threads, 3 CTAs/SM.  SPG_DENSE_CFG overrides.
// Segments the dense kernel caches next to a W-column panel within
// `smem_budget` (the per-segment panel offsets grow with the output width);
// < 32 means the geometry does not fit and the rows take the sort fallback.
template <int W, class SR, class Src>
int dense_seg_cap(int64_t ncols, size_t smem_budget, size_t* smem_out = nullptr) {
  using V = typename SR::value_type;
  const int64_t np64 = (ncols + W - 1) / W;
  if (np64 > (int64_t{1} << 20)) return 0;
  const int np = (int)np64;
  const bool preall = kPreAll && np <= 32;  // per-row prefixes of every panel (small panel counts)
  const size_t per_seg = SegCache<SR, Src>::bytes_per_seg(np) + (preall ? sizeof(int) * np : 0);
  const size_t fixed = sizeof(V) * W + sizeof(uint32_t) * (W / 32) + (preall ? sizeof(int) * (np + 4) : 0);
  const size_t room = smem_budget > fixed + 64 ? smem_budget - fixed - 64 : 0;
  const int cap = (int)std::min<size_t>(8192, room / per_seg) & ~3;  // keeps 16-byte values aligned
  if (smem_out) *smem_out = fixed + (size_t)cap * per_seg + 64;
  return cap;
}

template <int W, int DT, class SR, class Src, int MINB = 1>
void launch_dense_cfg(spg_ctx* c, cudaStream_t s, const Src& src, const int64_t* rows, int64_t n, int64_t ncols,
                      size_t smem_budget, unsigned long long* work, const RowOut<typename SR::value_type>& out) {
  const int np = (int)((ncols + W - 1) / W);
  const bool preall = kPreAll && np <= 32;
  size_t smem = 0;
  const int cap = dense_seg_cap<W, SR, Src>(ncols, smem_budget, &smem);
  if (cap < 32) fail(SPG_ERR_INTERNAL, "dense panel: no room for the segment cache");
  auto kern = dense_panel_kernel<SR, Src, W, DT, MINB>;
  set_smem(kern, smem);
  kern<<<resident_grid(c, kern, DT, smem, n), DT, smem, s>>>(src, rows, n, np, cap, work, out, preall);
  SPG_LAUNCH_CHECK();
  ++c->launches;
}

// Warp-specialised dense kernel: two W-column accumulators, PW product warps,
// EW emit warps, one CTA per SM.
template <int W, int PW, int EW, class SR, class Src>
void launch_dense_ws(spg_ctx* c, cudaStream_t s, const Src& src, const int64_t* rows, int64_t n, int64_t ncols,
                     size_t smem_budget, unsigned long long* work, const RowOut<typename SR::value_type>& out) {
  using V = typename SR::value_type;
  const int np = (int)((ncols + W - 1) / W);
  const size_t per_seg = SegCache<SR, Src>::bytes_per_seg(np);
  const size_t fixed = 2 * (sizeof(V) * W + sizeof(uint32_t) * (W / 32));
  const size_t room = smem_budget > fixed + 64 ? smem_budget - fixed - 64 : 0;
  const int cap = (int)std::min<size_t>(8192, room / per_seg) & ~3;
  if (cap < 32) fail(SPG_ERR_INTERNAL, "dense panel: no room for the segment cache");
  const size_t smem = fixed + (size_t)cap * per_seg + 64;
  auto kern = dense_panel_ws_kernel<SR, Src, W, PW, EW>;
  set_smem(kern, smem);
  kern<<<resident_grid(c, kern, (PW + EW) * 32, smem, n), (PW + EW) * 32, smem, s>>>(src, rows, n, np, cap, work,
                                                                                     out);
  SPG_LAUNCH_CHECK();
  ++c->launches;
}

inline int dense_cfg() {
  static int cfg = [] {
    const char* e = std::getenv("SPG_DENSE_CFG");
    return e ? std::atoi(e) : 1;
  }();
  return cfg;
}

template <class V>
inline int dense_panel_width() {
  const int cfg = dense_cfg();
  return Geom<V>::kPanelW >> (cfg == 1 || cfg == 7 ? 1 : 0);
}

template <class SR, class Src>
void launch_dense(spg_ctx* c, cudaStream_t s, const Src& src, const int64_t* rows, int64_t n, int64_t ncols,
                  unsigned long long* work, const RowOut<typename SR::value_type>& out) {
  using V = typename SR::value_type;
  constexpr int PW = Geom<V>::kPanelW;
  switch (dense_cfg()) {
    case 1:  // default: 64 KB panel, 512 threads, 2 CTAs/SM
      launch_dense_cfg<PW / 2, 512, SR, Src, 2>(c, s, src, rows, n, ncols, 110 * 1024, work, out);
      break;
    case 7:  // warp-specialised: 24 product + 8 emit warps, double-buffered 64 KB panels (measured slower)
      launch_dense_ws<PW / 2, 24, 8, SR, Src>(c, s, src, rows, n, ncols, 220 * 1024, work, out);
      break;
    default:  // 0: 128 KB panel, 1024 threads, 1 CTA/SM
      launch_dense_cfg<PW, 1024, SR, Src>(c, s, src, rows, n, ncols, 220 * 1024, work, out);
  }
}

// segment-cache capacity that fits next to a T-slot hash table
template <class V>
inline int V_hash_cap(int T) {
  const size_t table = (size_t)T * (sizeof(V) + 8);  // values + keys + staging
  const size_t room = table < 200 * 1024 ? 200 * 1024 - table : 0;
  const size_t per = 8 + 4 + sizeof(V) + 4 + 4;
  return (int)std::max<size_t>(64, std::min<size_t>(2048, room / per)) & ~3;
}

template <class SR>
inline void set_panels(MulSource<SR>& s, const int32_t* poff, int np, int) {
  s.poff = poff;
  s.npanels = np;
}
template <class SR>
inline void set_panels(MergeSource<SR>& s, const int32_t*, int, int w) {
  s.panel_w = w;
}
template <class SR>
inline bool needs_poff(const MulSource<SR>&) {
  return true;
}
template <class SR>
inline bool needs_poff(const MergeSource<SR>&) {
  return false;
}

#ifndef SPG_BITRANK_N
#define SPG_BITRANK_N 0  // bit-rank bin: rows with F <= this many products (0: 8192, 4096 for values > 4 B)
#endif

// Runs the pipeline for rows [0, src.nrows) with output width ncols_out.
// `r_for_panels` (the right operand) is needed to build the panel offsets
// of the dense bin for a MulSource.
template <class SR, class Src>
void run_rows(spg_ctx* c, const Src& src_in, int64_t ncols_out, spg_dcsr* out, spg_mult_stats* st,
              const spg_dcsr* r_for_panels = nullptr, bool* two_pass_out = nullptr) {
  using V = typename SR::value_type;
  const int64_t m = src_in.nrows;
  NvtxRange nv_all("spg:row pipeline (per-bin)");
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
  Src src = src_in;

  // K1 analyse
  DBuf<int64_t> prods(c, m), ub(c, m + 1), off(c, m + 1), rownnz(c, m + 1);
  DBuf<uint8_t> bins(c, m);
  static const int64_t dense_min = [] {  // SPG_DENSE_MIN: products above which a row goes dense
    const char* e = std::getenv("SPG_DENSE_MIN");
    return e ? (int64_t)std::atoll(e) : kDenseMinRow;
  }();
  // bit-rank bin (bin 8): rows with 512 < F <= kBitRankN whose output columns fit a window of 32*kBitRankW
  static const int bitrank_on = [] {
    const char* e = std::getenv("SPG_BITRANK");
    return e ? std::atoi(e) : 1;
  }();
  constexpr int kBitRankN = SPG_BITRANK_N > 0 ? SPG_BITRANK_N : (sizeof(V) <= 4 ? 8192 : 4096);
  constexpr int kBitRankW = 8192, kBitRankSegs = 256, kBitRankThreads = 512;
  // narrow outputs (<= 131072 columns): a half-size window when the full one would leave a single CTA per
  // SM (wide values; measured 8.1 -> 7.4 ms on ER max-times, no gain for 4-byte values at 2 CTAs/SM)
  constexpr int kBitRankW2 = 4096;
  auto br_bytes = [&](int w) {
    return sizeof(V) * kBitRankN + sizeof(uint32_t) * (w + w / 32) +
           sizeof(uint16_t) * (w + ((std::min(kBitRankN, w) + 7) & ~7)) +
           (size_t)kBitRankSegs * SegCache<SR, Src>::bytes_per_seg(1) + 64;
  };
  const size_t br_smem_wide = sizeof(V) * kBitRankN + sizeof(uint32_t) * (kBitRankW + kBitRankW / 32) +
                         sizeof(uint16_t) * (kBitRankW + ((kBitRankN + 7) & ~7)) +
                         (size_t)kBitRankSegs * SegCache<SR, Src>::bytes_per_seg(1) + 64;
  const bool br_narrow = ncols_out <= 32 * (int64_t)kBitRankW2 && br_smem_wide > 110 * 1024;
  const size_t br_smem = br_narrow ? br_bytes(kBitRankW2) : br_smem_wide;
  const bool bitrank = bitrank_on && !AddCanCancel<SR>::value && br_smem <= 220 * 1024;
  // rank-panel bin (bin 9): longer rows in the same window, accumulator panels in rank space
  static const int rankpanel_on = [] {
    const char* e = std::getenv("SPG_RANKPANEL");
    return e ? std::atoi(e) : 1;
  }();
  constexpr int kRpN = 65536 / (int)sizeof(V), kRpSegs = 1024, kRpThreads = 1024;
  const size_t rp_smem = sizeof(V) * kRpN + sizeof(uint32_t) * (kBitRankW + kBitRankW / 32) +
                         2 * sizeof(uint16_t) * kBitRankW + (sizeof(int64_t) + sizeof(int)) * kRpSegs +
                         (size_t)kRpSegs * SegCache<SR, Src>::bytes_per_seg(1) + 64;
  const bool rankpanel = bitrank && rankpanel_on && rp_smem <= 220 * 1024 && sizeof(V) == 4;  // measured gain: 4-byte values
  static const int64_t rp_maxf = [] {  // rank-panel rows: F up to this many products
    const char* e = std::getenv("SPG_RP_MAXF");
    return std::min<int64_t>(e ? (int64_t)std::atoll(e) : (int64_t)16384, 65535);  // 16-bit ranks
  }();
  DBuf<int32_t> colmin(c, bitrank ? (size_t)m : 1);
  analyse_rows_kernel<SR, Src><<<grid_for(c, m, 8), 256, 0, c->stream>>>(
      src, ncols_out, dense_min, bitrank ? kBitRankN : 0, kBitRankSegs, 32 * (int64_t)kBitRankW,  // window (both)
      rankpanel ? kRpSegs : 0, rp_maxf, 0, colmin.p, prods.p, ub.p, bins.p);
  SPG_LAUNCH_CHECK();
  ++c->launches;
  SPG_CUDA(cudaMemsetAsync(ub.p + m, 0, sizeof(int64_t), c->stream));
  SPG_CUDA(cudaMemsetAsync(rownnz.p + m, 0, sizeof(int64_t), c->stream));
  exclusive_scan(c, ub.p, off.p, m + 1);  // off[m] = total scratch entries
  DBuf<unsigned long long> counts(c, kNumBins + 1);
  SPG_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(unsigned long long) * (kNumBins + 1), c->stream));
  bin_count_kernel<<<grid_for(c, m, 1024, 2), 1024, 0, c->stream>>>(bins.p, m, counts.p);
  SPG_LAUNCH_CHECK();
  ++c->launches;
  unsigned long long hcounts[kNumBins];
  int64_t scratch_total = 0;
  SPG_CUDA(cudaMemcpyAsync(hcounts, counts.p, sizeof(hcounts), cudaMemcpyDeviceToHost, c->stream));
  SPG_CUDA(cudaMemcpyAsync(&scratch_total, off.p + m, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  {
    HostTrace ht("analyse sync");
    SPG_CUDA(cudaStreamSynchronize(c->stream));
  }
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
  // Dense-bin rows whose panel geometry does not fit next to the segment
  // cache (very wide outputs with wide values) take the sort fallback (bin 11).
  if (hcounts[kBinDense] > 0) {
    constexpr int PW = Geom<V>::kPanelW;
    const bool fits = dense_seg_cap<PW / 2, SR, Src>(ncols_out, 110 * 1024) >= 32 &&
                      dense_seg_cap<PW, SR, Src>(ncols_out, 220 * 1024) >= 32;
    if (!fits || c->pipeline == SPG_PIPE_SORTED) {
      relabel_bin_kernel<<<grid_for(c, m, 1024, 2), 1024, 0, c->stream>>>(bins.p, m, kBinDense, kBinWide);
      SPG_LAUNCH_CHECK();
      ++c->launches;
      hcounts[kBinWide] += hcounts[kBinDense];
      hcounts[kBinDense] = 0;
    }
  }

  // Panels for the dense bin.
  const int W = dense_panel_width<V>();
  const int np = npanels_for<V>(ncols_out, W);
  DBuf<int32_t> poff;
  if (hcounts[kBinDense] > 0 && np > 1) {
    if (needs_poff(src)) {
      if (!r_for_panels) fail(SPG_ERR_INTERNAL, "dense panels need the right operand");
      const spg_dcsr& R = *r_for_panels;
      poff = DBuf<int32_t>(c, (size_t)R.nrows * (np + 1));
      panel_offsets_kernel<<<grid_for(c, R.nrows, 8), 256, 0, c->stream>>>(R.nrows, R.ptr, R.idx, np, W, poff.p);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    set_panels(src, poff.p, np, W);
  }
  int end_bit = 0;
  while ((int64_t{1} << end_bit) < ncols_out) ++end_bit;

  // Output strategy.
  //  * sum U_i entries fit the budget: each row writes into its own U_i slot
  //    of the scratch (direct placement at the U prefix), then a streaming
  //    compaction copies the exact rows into C;
  //  * otherwise exact-claim mode: each row (dense rows: each panel chunk)
  //    claims exactly its nnz in a scratch of `budget` bytes, then the
  //    compaction gathers the rows into C in row order;
  //  * if even the claims overflow (C too large to sit in HBM twice), that
  //    pass has still produced the exact rowptr: C is allocated once and the
  //    same kernels run again writing straight into it.
  size_t budget = c->scratch_budget;
  if (budget == 0) budget = (size_t)(mem_available(c) * 0.45);
  const size_t per_entry = sizeof(int32_t) + sizeof(V);
  int64_t cap = std::min<int64_t>(scratch_total, (int64_t)(budget / per_entry));
  DBuf<int32_t> sc_cols;
  DBuf<V> sc_vals;
  while (cap > 0) {  // the estimate can be stale (other allocators): shrink on OOM
    int32_t* pc = try_dalloc<int32_t>(c, (size_t)cap + 16);  // slack: vector reads may pass a row end
    V* pv = pc ? try_dalloc<V>(c, (size_t)cap + 16) : nullptr;
    if (pv) {
      sc_cols = DBuf<int32_t>::adopt(c, pc, (size_t)cap);
      sc_vals = DBuf<V>::adopt(c, pv, (size_t)cap);
      break;
    }
    if (pc) dfree(c, pc);
    mem_snapshot(c);
    cap = cap < (int64_t{1} << 20) ? 0 : cap / 2;
  }
  const int npc = std::max(np, 1);
  const bool slotted = cap > 0 && cap == scratch_total;  // U_i slots: no claims needed
  // U-slot mode: dense rows emit per-warp chunks (no block scan per panel)
  static const int warp_emit_on = [] {
    const char* e = std::getenv("SPG_WARP_EMIT");
    return e ? std::atoi(e) : 1;
  }();
  const bool warp_emit = warp_emit_on && slotted && hcounts[kBinDense] > 0 && dense_cfg() == 1;
  // chunks per dense slot: panels x warps of the 2-CTA kernel (W/2 panels, 16
  // warps) and of the heavy-row kernel (W panels, 32 warps) — they differ when
  // ncols is not a multiple of W (e.g. ncols <= W/2), so take the larger
  const int wstride = std::max(npc * (512 / 32), std::max(npanels_for<V>(ncols_out, Geom<V>::kPanelW), 1) * (1024 / 32));
  DBuf<int32_t> wchunks(c, warp_emit ? (size_t)hcounts[kBinDense] * wstride * 2 : 1);
  if (warp_emit)  // the 2-CTA rows fill fewer chunks than the stride holds: the rest must read as empty
    SPG_CUDA(cudaMemsetAsync(wchunks.p, 0, sizeof(int32_t) * hcounts[kBinDense] * wstride * 2, c->stream));
  DBuf<int64_t> rowstart, chunks;
  DBuf<unsigned long long> bump(c, 1);
  if (cap > 0 && !slotted) {
    rowstart = DBuf<int64_t>(c, (size_t)m);
    if (hcounts[kBinDense] > 0) {
      chunks = DBuf<int64_t>(c, (size_t)hcounts[kBinDense] * npc * 2);
      SPG_CUDA(cudaMemsetAsync(chunks.p, 0, sizeof(int64_t) * hcounts[kBinDense] * npc * 2, c->stream));
    }
    SPG_CUDA(cudaMemsetAsync(bump.p, 0, sizeof(unsigned long long), c->stream));
  }
  tm.mark(1);

  DBuf<int64_t> lists(c, m);
  DBuf<unsigned long long> cursor(c, kNumBins);
  unsigned long long base[kNumBins];
  {
    unsigned long long acc = 0;
    for (int b = 0; b < kNumBins; ++b) {
      base[b] = acc;
      if (b > 0) acc += hcounts[b];
    }
  }
  SPG_CUDA(cudaMemcpyAsync(cursor.p, base, sizeof(base), cudaMemcpyHostToDevice, c->stream));
  bin_scatter_kernel<<<grid_for(c, m, 1024, 2), 1024, 0, c->stream>>>(bins.p, m, cursor.p, lists.p);
  SPG_LAUNCH_CHECK();
  ++c->launches;
  // Row order inside each bin: the scatter's block arrival order scatters a
  // bin's rows over ~300K-row spans, while neighbouring rows of A usually
  // share right-operand rows — CTAs on nearby rows keep those in L2
  // (27-point stencil: the right operand's rows i +- N^2 stay resident).
  if (m >= 65536) {
    int row_bits = 1;
    while ((int64_t{1} << row_bits) < m) ++row_bits;
    DBuf<int64_t> alt(c, m);
    for (int b = 1; b < kNumBins; ++b) {
      const int64_t nbin = (int64_t)hcounts[b];
      if (b == kBinDense || nbin < 2) continue;  // dense rows are ordered by F below
      cub::DoubleBuffer<int64_t> db(lists.p + base[b], alt.p + base[b]);
      size_t bytes = 0;
      SPG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, db, (int)nbin, 0, row_bits, c->stream));
      ensure_cub_tmp(c, bytes);
      SPG_CUDA(cub::DeviceRadixSort::SortKeys(c->cub_tmp, bytes, db, (int)nbin, 0, row_bits, c->stream));
      ++c->launches;
      if (db.Current() != lists.p + base[b])
        SPG_CUDA(cudaMemcpyAsync(lists.p + base[b], db.Current(), sizeof(int64_t) * nbin, cudaMemcpyDeviceToDevice,
                                 c->stream));
    }
  }
  // dense bin: largest rows first
  const int64_t nd = (int64_t)hcounts[kBinDense];
  const int64_t* dense_rows = lists.p + base[kBinDense];
  DBuf<int64_t> dense_sorted, dk1, dk2;
  if (nd > 1) {
    dk1 = DBuf<int64_t>(c, nd);
    dk2 = DBuf<int64_t>(c, nd);
    dense_sorted = DBuf<int64_t>(c, nd);
    gather_keys_kernel<<<grid_for(c, nd, 256, 4), 256, 0, c->stream>>>(dense_rows, nd, prods.p, dk1.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
    size_t bytes = 0;
    SPG_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, dk1.p, dk2.p, dense_rows, dense_sorted.p,
                                                        (int)nd, 0, 64, c->stream));
    ensure_cub_tmp(c, bytes);
    SPG_CUDA(cub::DeviceRadixSort::SortPairsDescending(c->cub_tmp, bytes, dk1.p, dk2.p, dense_rows, dense_sorted.p,
                                                        (int)nd, 0, 64, c->stream));
    ++c->launches;
    dense_rows = dense_sorted.p;
  }
  // Heavy dense rows (F > kHeavyF: hundreds to thousands of segments) run in
  // a 1-CTA/SM kernel with twice the panel width and a ~1000-segment cache
  // (no segment batching); measured 2.2x faster for them than the 2-CTA one.
  constexpr int64_t kHeavyF = 262144;
  int64_t nh = 0;
  Src src_heavy = src;
  DBuf<int32_t> poff_heavy;
  static const int heavy_on = [] {
    const char* e = std::getenv("SPG_DENSE_HEAVY");
    return e ? std::atoi(e) : 1;
  }();
  if (heavy_on && nd > 0 && dense_cfg() == 1) {
    DBuf<unsigned long long> cnt(c, 1);
    SPG_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), c->stream));
    count_above_kernel<<<grid_for(c, nd, 256, 2), 256, 0, c->stream>>>(dense_rows, nd, prods.p, kHeavyF, cnt.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
    nh = (int64_t)d2h_scalar(c, cnt.p);
    if (nh > 0) {
      const int W2 = Geom<V>::kPanelW;
      const int np2 = npanels_for<V>(ncols_out, W2);
      if (np2 > 1 && needs_poff(src)) {
        const spg_dcsr& R = *r_for_panels;
        poff_heavy = DBuf<int32_t>(c, (size_t)R.nrows * (np2 + 1));
        panel_offsets_kernel<<<grid_for(c, R.nrows, 8), 256, 0, c->stream>>>(R.nrows, R.ptr, R.idx, np2, W2,
                                                                            poff_heavy.p);
        SPG_LAUNCH_CHECK();
        ++c->launches;
      }
      set_panels(src_heavy, poff_heavy.p, np2, W2);
    }
  }
  if (hcounts[kBinEmpty] > 0) {
    zero_empty_rows_kernel<<<grid_for(c, m, 256, 4), 256, 0, c->stream>>>(bins.p, m, rownnz.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
  }
  DBuf<unsigned long long> work(c, 2);
  float ms_numeric = 0.f, ms_compact = 0.f;
  // 2K-slot hash rows (512 < F <= 1024) are first tried in a 512-slot table
  // (many CTAs per SM, 4x fewer slots to clear and scan); rows with more than
  // 256 distinct columns are re-run in the 2K table (SPG_HASH_OPT=0: off)
  static const int hash_opt_on = [] {
    const char* e = std::getenv("SPG_HASH_OPT");
    return e ? std::atoi(e) : 1;
  }();
  const bool hash_opt = hash_opt_on && hcounts[kBinHash2K] > 0;
  DBuf<unsigned long long> ovf_n(c, 1);
  DBuf<int64_t> ovf_rows(c, hash_opt ? (size_t)hcounts[kBinHash2K] : 1);
  // global value tables for the 512- / 2K-slot hash bins (fp64 +): zeroed
  // once, left zero by every launch
  DBuf<V> gtab;
  size_t gtab_slots = 0;
  static const int gred_env = [] {
    const char* e = std::getenv("SPG_HASH_GRED");
    return e ? std::atoi(e) : 0;
  }();
  if (has_red_global<SR>::value && gred_env && hcounts[kBinHash2K] > 0) {
    gtab_slots = (size_t)c->sm_count * 16 * 2048;
    gtab = DBuf<V>(c, gtab_slots);
    SPG_CUDA(cudaMemsetAsync(gtab.p, 0, sizeof(V) * gtab_slots, c->stream));
  }

  // One numeric pass over all bins with output placement `o`.
  auto numeric = [&](const RowOut<V>& o) {
    SPG_CUDA(cudaMemsetAsync(work.p, 0, 2 * sizeof(unsigned long long), c->stream));
    if (hash_opt) SPG_CUDA(cudaMemsetAsync(ovf_n.p, 0, sizeof(unsigned long long), c->stream));
    const int64_t* lb = lists.p;
    StreamFork fk(c, 3);
    static const int plan = [] {  // SPG_STREAM_PLAN (default 1): heavy rows and rank panels on their own streams
      const char* e = std::getenv("SPG_STREAM_PLAN");
      return e ? std::atoi(e) : 1;
    }();
    if (nh > 0) {
      constexpr int PW = Geom<V>::kPanelW;
      launch_dense_cfg<PW, 1024, SR, Src>(c, plan == 1 ? fk[1] : fk[0], src_heavy, dense_rows, nh, ncols_out,
                                          220 * 1024, work.p + 1, o);
    }
    if (nd > nh) {
      RowOut<V> rest = o;
      rest.slot_base = nh;
      launch_dense<SR, Src>(c, fk[0], src, dense_rows + nh, nd - nh, ncols_out, work.p, rest);
    }
    if (hcounts[kBinHashMax] > 0)
      launch_hash<SR, Src, Geom<V>::kMaxT, 1024>(c, fk[1], src, lb + base[kBinHashMax], hcounts[kBinHashMax],
                                                 V_hash_cap<V>(Geom<V>::kMaxT), end_bit, o);
    if (hcounts[kBinHash8K] > 0)
      launch_hash<SR, Src, 8192, 512>(c, fk[1], src, lb + base[kBinHash8K], hcounts[kBinHash8K], 256, end_bit, o);
    if (hcounts[kBinHash4K] > 0)
      launch_hash<SR, Src, 4096, 256>(c, fk[2], src, lb + base[kBinHash4K], hcounts[kBinHash4K], 256, end_bit, o);
    if (hash_opt)
      launch_hash<SR, Src, 512, 128, true>(c, fk[2], src, lb + base[kBinHash2K], hcounts[kBinHash2K], 64, end_bit, o,
                                           ovf_n.p, ovf_rows.p, gtab.p, gtab_slots);
    else if (hcounts[kBinHash2K] > 0)
      launch_hash<SR, Src, 2048, 128>(c, fk[2], src, lb + base[kBinHash2K], hcounts[kBinHash2K], 256, end_bit, o,
                                      nullptr, nullptr, gtab.p, gtab_slots);
    if (hcounts[kBinEsc512] > 0)
      launch_esc<SR, Src, 128, 4>(c, fk[2], src, lb + base[kBinEsc512], hcounts[kBinEsc512], end_bit, o);
    if (hcounts[kBinBitRank] > 0) {
      if (br_narrow) {  // ncols <= 32*W2: every window fits the half-size bitmap
        auto kern = bitrank_rows_kernel<SR, Src, kBitRankThreads, kBitRankN, kBitRankW2>;
        set_smem(kern, br_smem);
        kern<<<resident_grid(c, kern, kBitRankThreads, br_smem, (int64_t)hcounts[kBinBitRank]), kBitRankThreads,
               br_smem, fk[1]>>>(src, lb + base[kBinBitRank], (int64_t)hcounts[kBinBitRank], kBitRankSegs, colmin.p, o);
      } else {
        auto kern = bitrank_rows_kernel<SR, Src, kBitRankThreads, kBitRankN, kBitRankW>;
        set_smem(kern, br_smem);
        kern<<<resident_grid(c, kern, kBitRankThreads, br_smem, (int64_t)hcounts[kBinBitRank]), kBitRankThreads,
               br_smem, fk[1]>>>(src, lb + base[kBinBitRank], (int64_t)hcounts[kBinBitRank], kBitRankSegs, colmin.p, o);
      }
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    if (hcounts[kBinRankPanels] > 0) {
      auto kern = rankpanel_rows_kernel<SR, Src, kRpThreads, kRpN, kBitRankW>;
      set_smem(kern, rp_smem);
      kern<<<resident_grid(c, kern, kRpThreads, rp_smem, (int64_t)hcounts[kBinRankPanels]), kRpThreads, rp_smem,
             plan == 1 ? fk[2] : fk[0]>>>(src, lb + base[kBinRankPanels], (int64_t)hcounts[kBinRankPanels], kRpSegs,
                                          colmin.p, o);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    if (hcounts[kBinWarpEsc] > 0) {
      esc_warp_kernel<SR, Src><<<grid_for(c, hcounts[kBinWarpEsc], 8), 256, 0, fk[2]>>>(
          src, lb + base[kBinWarpEsc], hcounts[kBinWarpEsc], o);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    fk.join();
    if (hash_opt) {  // the rows that overflowed the 512-slot table
      const int64_t nov = (int64_t)d2h_scalar(c, ovf_n.p);
      if (nov > 0)
        launch_hash<SR, Src, 2048, 128>(c, c->stream, src, ovf_rows.p, nov, 256, end_bit, o, nullptr, nullptr, gtab.p,
                                        gtab_slots);
    }
    if (hcounts[kBinWide] > 0)
      run_wide_rows<SR, Src>(c, src, lb + base[kBinWide], (int64_t)hcounts[kBinWide], prods.p, o);
  };

  RowOut<V> first;
  first.rownnz = rownnz.p;
  if (cap > 0) {
    first.cols = sc_cols.p;
    first.vals = sc_vals.p;
    if (slotted) {
      first.off = off.p;
      if (warp_emit) {
        first.wchunks = wchunks.p;
        first.wstride = wstride;
      }
    } else {
      first.bump = bump.p;
      first.cap = cap;
      first.rowstart = rowstart.p;
      first.chunks = chunks.p;
      first.chunk_stride = npc;
    }
  }
  numeric(first);
  exclusive_scan(c, rownnz.p, out->ptr, m + 1);
  const int64_t nnz = d2h_scalar(c, out->ptr + m);
  const unsigned long long claimed = cap > 0 && !slotted ? d2h_scalar(c, bump.p) : 0ull;
  const bool fits = slotted || (cap > 0 && (int64_t)claimed <= cap);
  tm.mark(2);
  ms_numeric = tm.between(1, 2);
  if (!fits) {  // second pass straight into C (the scratch is released first)
    sc_cols.reset();
    sc_vals.reset();
  }
  out->nnz = nnz;
  out->idx = dalloc<int32_t>(c, (size_t)nnz);
  out->vals = dalloc<V>(c, (size_t)nnz);
  if (fits) {
    constexpr bool kWords = sizeof(V) % 4 == 0;
    const bool long_rows = kWords && slotted && nd > 0 && !warp_emit;  // dense rows: CTA per row, 16-byte copies
    compact_rows_kernel<V><<<grid_for(c, m, 8), 256, 0, c->stream>>>(
        m, (long_rows || warp_emit) ? bins.p : nullptr, slotted ? off.p : rowstart.p, out->ptr, sc_cols.p, sc_vals.p,
        out->idx, static_cast<V*>(out->vals));
    SPG_LAUNCH_CHECK();
    ++c->launches;
    if (warp_emit) {
      compact_wchunks_kernel<V, 256><<<grid_for(c, nd, 1, 8), 256, 0, c->stream>>>(
          dense_rows, nd, wchunks.p, wstride, off.p, out->ptr, sc_cols.p, sc_vals.p, out->idx,
          static_cast<V*>(out->vals));
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    if constexpr (kWords) {
      if (long_rows) {
        compact_long_rows_kernel<V><<<grid_for(c, nd, 1, 8), 256, 0, c->stream>>>(
            dense_rows, nd, off.p, out->ptr, sc_cols.p, sc_vals.p, out->idx, static_cast<V*>(out->vals));
        SPG_LAUNCH_CHECK();
        ++c->launches;
      }
    }
    if (nd > 0 && !slotted) {
      compact_chunks_kernel<V><<<grid_for(c, nd, 1, 8), 256, 0, c->stream>>>(
          dense_rows, nd, npc, chunks.p, out->ptr, sc_cols.p, sc_vals.p, out->idx, static_cast<V*>(out->vals));
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    sc_cols.reset();
    sc_vals.reset();
    tm.mark(3);
    ms_compact = tm.between(2, 3);
  } else {
    RowOut<V> direct;
    direct.cols = out->idx;
    direct.vals = static_cast<V*>(out->vals);
    direct.off = out->ptr;
    direct.rownnz = rownnz.p;
    numeric(direct);
    tm.mark(3);
    ms_numeric += tm.between(2, 3);
  }
  if (two_pass_out) *two_pass_out = !fits;
  if (HostTrace::limit_ms() >= 0)
    std::fprintf(stderr, "[spg-host] rows=%lld U=%lld cap=%lld nnz=%lld claimed=%llu budget=%zu mode=%d\n",
                 (long long)m, (long long)scratch_total, (long long)cap, (long long)nnz, claimed, budget,
                 !fits ? 2 : slotted ? 0 : 1);
  if (st) {
    tm.mark(3);
    st->products = products;
    st->nnz_out = out->nnz;
    for (int b = 0; b < kNumBins; ++b) st->rows_per_bin[b] = (int64_t)hcounts[b];
    st->ms_numeric = ms_numeric;
    st->ms_compact = ms_compact;
    st->ms_total = tm.between(0, 3);
    st->ms_analyse = st->ms_total - ms_numeric - ms_compact;
    st->kernels = (int64_t)(c->launches - launches0);
    st->output_mode = !fits ? 2 : slotted ? 0 : 1;
  }
}


// ---------------------------------------------------------------------------
// Bitmap-rank driver (bitmap_rank.cuh) for a local multiply whose output
// width fits a shared-memory bitmap: rows with F > SPG_BR_MINF products take
// the symbolic-bitmap / rank path and write straight into C; the short rows
// run the hash / ESC kernels into U-slot scratch and only they are compacted.
// Returns false (nothing changed) when the call is not eligible or the
// bitmaps do not fit the memory budget; the caller then runs run_rows.
// ---------------------------------------------------------------------------
template <class SR>
bool run_rows_br(spg_ctx* c, const MulSource<SR>& src, const spg_dcsr* r, int64_t ncols_out, spg_dcsr* out,
                 spg_mult_stats* st) {
  using V = typename SR::value_type;
  using Src = MulSource<SR>;
  static const int br_on = [] {
    const char* e = std::getenv("SPG_BR");
    return e ? std::atoi(e) : 1;
  }();
  static const int64_t br_minf = [] {  // rows with more products take the bitmap path (<= 4096: see below)
    const char* e = std::getenv("SPG_BR_MINF");
    return std::min<int64_t>(e ? (int64_t)std::atoll(e) : 2048, 4096);
  }();
  const int64_t m = src.nrows;
  if (!br_on || c->pipeline != SPG_PIPE_AUTO || m == 0 || ncols_out <= 0 || ncols_out > kBrMaxCols)
    return false;
  const int64_t nnz_r = r->nnz;
  if (nnz_r >= (int64_t{1} << 31) - 64) return false;  // 32-bit entry offsets
  const int nwords = br_words(ncols_out);
  PhaseTimer tm(c, st != nullptr);
  const uint64_t launches0 = c->launches;
  tm.mark(0);

  NvtxRange nv_all("spg:local_multiply (bitmap-rank)");
  // K1 analyse: F <= br_minf (<= 4096) rows go to the ESC / hash bins only
  DBuf<int64_t> prods(c, m), ub(c, m + 1), off(c, m + 1), rownnz(c, m + 1);
  DBuf<uint8_t> bins(c, m);
  DBuf<int32_t> colmin(c, 1);
  analyse_rows_kernel<SR, Src><<<grid_for(c, m, 8), 256, 0, c->stream>>>(
      src, ncols_out, INT64_MAX, 0, 0, 0, 0, 0, br_minf, colmin.p, prods.p, ub.p, bins.p);
  SPG_LAUNCH_CHECK();
  ++c->launches;
  SPG_CUDA(cudaMemsetAsync(ub.p + m, 0, sizeof(int64_t), c->stream));
  SPG_CUDA(cudaMemsetAsync(rownnz.p + m, 0, sizeof(int64_t), c->stream));
  exclusive_scan(c, ub.p, off.p, m + 1);
  DBuf<unsigned long long> counts(c, kNumBins + 1);
  SPG_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(unsigned long long) * (kNumBins + 1), c->stream));
  bin_count_kernel<<<grid_for(c, m, 1024, 2), 1024, 0, c->stream>>>(bins.p, m, counts.p);
  SPG_LAUNCH_CHECK();
  ++c->launches;
  unsigned long long hcounts[kNumBins];
  int64_t scratch_total = 0;
  SPG_CUDA(cudaMemcpyAsync(hcounts, counts.p, sizeof(hcounts), cudaMemcpyDeviceToHost, c->stream));
  SPG_CUDA(cudaMemcpyAsync(&scratch_total, off.p + m, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  SPG_CUDA(cudaStreamSynchronize(c->stream));
  const int64_t nb = (int64_t)hcounts[kBinBitmap];

  // memory: U-slot scratch of the short rows + one bitmap per long row
  size_t budget = c->scratch_budget;
  if (budget == 0) budget = (size_t)(mem_available(c) * 0.45);
  const size_t bm_bytes = (size_t)nb * nwords * sizeof(uint32_t);
  const size_t sc_bytes = (size_t)scratch_total * (sizeof(int32_t) + sizeof(V));
  if (bm_bytes + sc_bytes > budget) return false;
  uint32_t* gbm_p = nb > 0 ? try_dalloc<uint32_t>(c, (size_t)nb * nwords) : nullptr;
  if (nb > 0 && !gbm_p) return false;
  DBuf<uint32_t> gbm = DBuf<uint32_t>::adopt(c, gbm_p, (size_t)nb * nwords);
  DBuf<int32_t> sc_cols(c, (size_t)scratch_total + 16);
  DBuf<V> sc_vals(c, (size_t)scratch_total + 16);

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
  int end_bit = 0;
  while ((int64_t{1} << end_bit) < ncols_out) ++end_bit;

  // K2 bin lists; the bitmap bin sorted by F descending (largest rows first)
  DBuf<int64_t> lists(c, m);
  DBuf<unsigned long long> cursor(c, kNumBins);
  unsigned long long base[kNumBins];
  {
    unsigned long long acc = 0;
    for (int b = 0; b < kNumBins; ++b) {
      base[b] = acc;
      if (b > 0) acc += hcounts[b];
    }
  }
  SPG_CUDA(cudaMemcpyAsync(cursor.p, base, sizeof(base), cudaMemcpyHostToDevice, c->stream));
  bin_scatter_kernel<<<grid_for(c, m, 1024, 2), 1024, 0, c->stream>>>(bins.p, m, cursor.p, lists.p);
  SPG_LAUNCH_CHECK();
  ++c->launches;
  const int64_t* brows = lists.p + base[kBinBitmap];
  DBuf<int64_t> bsorted, bk1, bk2;
  if (nb > 1) {
    bk1 = DBuf<int64_t>(c, nb);
    bk2 = DBuf<int64_t>(c, nb);
    bsorted = DBuf<int64_t>(c, nb);
    gather_keys_kernel<<<grid_for(c, nb, 256, 4), 256, 0, c->stream>>>(brows, nb, prods.p, bk1.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
    size_t bytes = 0;
    SPG_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, bk1.p, bk2.p, brows, bsorted.p, (int)nb, 0,
                                                        64, c->stream));
    ensure_cub_tmp(c, bytes);
    SPG_CUDA(cub::DeviceRadixSort::SortPairsDescending(c->cub_tmp, bytes, bk1.p, bk2.p, brows, bsorted.p, (int)nb,
                                                        0, 64, c->stream));
    ++c->launches;
    brows = bsorted.p;
  }
  if (hcounts[kBinEmpty] > 0) {
    zero_empty_rows_kernel<<<grid_for(c, m, 256, 4), 256, 0, c->stream>>>(bins.p, m, rownnz.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
  }
  DBuf<unsigned long long> work(c, 2);
  SPG_CUDA(cudaMemsetAsync(work.p, 0, 2 * sizeof(unsigned long long), c->stream));
  tm.mark(1);

#ifndef SPG_BR_NUM_THREADS
#define SPG_BR_NUM_THREADS 512  // fold CTA size
#endif
#ifndef SPG_BR_NUM_CTAS
#define SPG_BR_NUM_CTAS 2  // fold CTAs per SM (shared memory split between them)
#endif
  constexpr int kSymThreads = 512, kNumThreads = SPG_BR_NUM_THREADS;
  // numeric geometry: 2 CTAs/SM when the bitmap is <= 32 KB, else 1; the rest
  // of the CTA's shared memory is the rank window's accumulator
  auto num_kern = br_numeric_kernel<SR, Src, kNumThreads, SPG_BR_NUM_CTAS>;
  int capv = 0;
  {
    cudaFuncAttributes fa{};
    SPG_CUDA(cudaFuncGetAttributes(&fa, num_kern));
    const size_t per_sm = 232448 - 2048;  // usable shared memory per SM, 1 KB reserved per CTA
    const size_t num_budget = (nwords <= 8192 ? per_sm / SPG_BR_NUM_CTAS : per_sm) - fa.sharedSizeBytes - 256;
    const BrNumLayout<V> l0{nwords + 8, 0};
    const size_t fixed = l0.bytes(kNumThreads);
    capv = fixed < num_budget ? (int)std::min<size_t>(65535, (num_budget - fixed) / sizeof(V)) & ~7 : 0;
    if (capv < 1024) fail(SPG_ERR_INTERNAL, "bitmap-rank: no shared memory left for the accumulator");
  }
  // fine column panels: window boundaries fall on them, so a segment's slice
  // of a window comes from the right operand's panel offsets (no search)
  int wf = 1024;  // panel width: ~64 panels per row (<= kBrMaxPanels; a panel never exceeds capv outputs)
  while ((ncols_out + wf - 1) / wf > kBrMaxPanels) wf *= 2;
  while (wf * 2 <= capv && (ncols_out + wf - 1) / wf > 64) wf *= 2;
  if (wf > capv || wf / 32 > 32 * (nwords / kSymThreads)) return false;
  const int npf = (int)((ncols_out + wf - 1) / wf);
  const int wpp = wf / 32;
  const int wstride = npf + 2;
  DBuf<int2> wlist(c, (size_t)std::max<int64_t>(nb, 1) * wstride);
  DBuf<int32_t> nwin(c, (size_t)nb + 1);
  DBuf<int32_t> poff;
  if (nb > 0) {
    poff = DBuf<int32_t>(c, (size_t)r->nrows * (npf + 1));
    panel_offsets_kernel<<<grid_for(c, r->nrows, 8), 256, 0, c->stream>>>(r->nrows, r->ptr, r->idx, npf, wf, poff.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
  }
  {  // symbolic (long rows) || numeric of the short rows into their slots
    NvtxRange nv("spg:symbolic bitmaps + short rows");
    StreamFork fk(c, 3);
    if (nb > 0) {
      const size_t smem = sizeof(uint32_t) * (size_t)nwords + BrSegs<V>::bytes(kSymThreads) + 64;
      auto kern = br_symbolic_kernel<SR, Src, kSymThreads, SPG_BR_SYM_MINB>;
      set_smem(kern, smem);
      kern<<<resident_grid(c, kern, kSymThreads, smem, nb), kSymThreads, smem, fk[0]>>>(
          src, brows, nb, nwords, capv, wpp, npf, wstride, work.p, gbm.p, wlist.p, nwin.p, rownnz.p);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    RowOut<V> o;
    o.cols = sc_cols.p;
    o.vals = sc_vals.p;
    o.off = off.p;
    o.rownnz = rownnz.p;
    const int64_t* lb = lists.p;
    if (hcounts[kBinHash8K] > 0)
      launch_hash<SR, Src, 8192, 512>(c, fk[1], src, lb + base[kBinHash8K], hcounts[kBinHash8K], 256, end_bit, o);
    if (hcounts[kBinHash4K] > 0)
      launch_hash<SR, Src, 4096, 256>(c, fk[1], src, lb + base[kBinHash4K], hcounts[kBinHash4K], 256, end_bit, o);
    if (hcounts[kBinHash2K] > 0)
      launch_hash<SR, Src, 2048, 128>(c, fk[2], src, lb + base[kBinHash2K], hcounts[kBinHash2K], 256, end_bit, o);
    if (hcounts[kBinEsc512] > 0)
      launch_esc<SR, Src, 128, 4>(c, fk[2], src, lb + base[kBinEsc512], hcounts[kBinEsc512], end_bit, o);
    if (hcounts[kBinWarpEsc] > 0) {
      esc_warp_kernel<SR, Src><<<grid_for(c, hcounts[kBinWarpEsc], 8), 256, 0, fk[2]>>>(
          src, lb + base[kBinWarpEsc], hcounts[kBinWarpEsc], o);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    for (int b : {(int)kBinDense, (int)kBinHashMax, (int)kBinBitRank, (int)kBinRankPanels})
      if (hcounts[b] > 0) fail(SPG_ERR_INTERNAL, "bitmap-rank driver: unexpected bin");
    fk.join();
  }
  out->ptr = dalloc<int64_t>(c, m + 1);
  exclusive_scan(c, rownnz.p, out->ptr, m + 1);
  // (row, window) work items
  DBuf<int64_t> winoff(c, (size_t)nb + 1);
  DBuf<int2> items;
  int64_t nitems = 0;
  if (nb > 0) {
    DBuf<int64_t> nwin64(c, (size_t)nb + 1);
    widen_kernel<<<grid_for(c, nb + 1, 256, 4), 256, 0, c->stream>>>(nwin.p, nb, nwin64.p);
    SPG_LAUNCH_CHECK();
    exclusive_scan(c, nwin64.p, winoff.p, nb + 1);
    c->launches += 1;
  }
  int64_t hv[2] = {0, 0};
  SPG_CUDA(cudaMemcpyAsync(&hv[0], out->ptr + m, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  if (nb > 0) SPG_CUDA(cudaMemcpyAsync(&hv[1], winoff.p + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  SPG_CUDA(cudaStreamSynchronize(c->stream));
  const int64_t nnz = hv[0];
  nitems = hv[1];
  bool r_small = false;
  if constexpr (has_mul_small<SR>::value) {
    if (nitems > 0) {
      DBuf<unsigned long long> ns(c, 1);
      SPG_CUDA(cudaMemsetAsync(ns.p, 0, sizeof(unsigned long long), c->stream));
      br_count_not_small_kernel<SR><<<grid_for(c, nnz_r, 256, 8), 256, 0, c->stream>>>(nnz_r, src.rval, ns.p);
      SPG_LAUNCH_CHECK();
      ++c->launches;
      r_small = d2h_scalar(c, ns.p) == 0;
    }
  }
  DBuf<BrPack<V>> pack;
  if constexpr (sizeof(V) <= 8) {
    if (nitems > 0 && nnz_r > 0) {
      pack = DBuf<BrPack<V>>(c, (size_t)nnz_r);
      br_pack_kernel<V><<<grid_for(c, nnz_r, 256, 8), 256, 0, c->stream>>>(nnz_r, src.ridx, src.rval, pack.p);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
  }
  if (nitems > 0) {
    items = DBuf<int2>(c, (size_t)nitems);
    br_expand_items_kernel<<<grid_for(c, nb, 256, 4), 256, 0, c->stream>>>(nb, nwin.p, winoff.p, items.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
  }
  tm.mark(2);
  const float ms_sym = tm.between(1, 2);
  out->nrows = m;
  out->ncols = ncols_out;
  out->nnz = nnz;
  out->idx = dalloc<int32_t>(c, (size_t)nnz);
  out->vals = dalloc<V>(c, (size_t)nnz);
  DBuf<unsigned long long> zeros(c, 1);
  DBuf<unsigned long long> rowzero(c, (size_t)m);
  SPG_CUDA(cudaMemsetAsync(zeros.p, 0, sizeof(unsigned long long), c->stream));
  SPG_CUDA(cudaMemsetAsync(rowzero.p, 0, sizeof(unsigned long long) * (size_t)m, c->stream));
  {  // numeric (long rows, straight into C) || compaction of the short rows
    NvtxRange nv("spg:rank-space fold + short-row compaction");
    StreamFork fk(c, 2);
    if (nitems > 0) {
      const size_t smem = BrNumLayout<V>{nwords + 8, capv}.bytes(kNumThreads);
      auto kern = num_kern;
      set_smem(kern, smem);
      kern<<<resident_grid(c, kern, kNumThreads, smem, nitems), kNumThreads, smem, fk[0]>>>(
          src, pack.p, items.p, nitems, brows, ncols_out, nwords, capv, wpp, npf, wstride, wlist.p, poff.p, r_small, work.p + 1,
          gbm.p, out->ptr,
          out->idx, static_cast<V*>(out->vals), zeros.p, rowzero.p);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    if (scratch_total > 0) {
      compact_rows_kernel<V><<<grid_for(c, m, 8), 256, 0, fk[1]>>>(m, bins.p, off.p, out->ptr, sc_cols.p, sc_vals.p,
                                                                 out->idx, static_cast<V*>(out->vals));
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    fk.join();
  }
  tm.mark(3);
  const float ms_num = tm.between(2, 3);
#ifdef SPG_BR_PROF
  {
    unsigned long long pr[16];
    SPG_CUDA(cudaMemcpyFromSymbol(pr, br_prof, sizeof(pr)));
    const unsigned long long z[16] = {};
    SPG_CUDA(cudaMemcpyToSymbol(br_prof, z, sizeof(z)));
    std::fprintf(stderr, "[br-prof] items=%lld rows=%lld cycles(G):", (long long)nitems, (long long)nb);
    for (int k = 0; k < 12; ++k) std::fprintf(stderr, " %d:%.3f", k, pr[k] * 1e-9);
    std::fprintf(stderr, "\n");
  }
#endif
  gbm.reset();
  sc_cols.reset();
  sc_vals.reset();
  if (nb > 0 && d2h_scalar(c, zeros.p) > 0) {  // entries that folded to zero(): drop them
    DBuf<int64_t> kept(c, (size_t)m + 1), nptr(c, (size_t)m + 1);
    br_kept_counts_kernel<<<grid_for(c, m, 256, 4), 256, 0, c->stream>>>(m, out->ptr, rowzero.p, kept.p);
    SPG_LAUNCH_CHECK();
    SPG_CUDA(cudaMemsetAsync(kept.p + m, 0, sizeof(int64_t), c->stream));
    exclusive_scan(c, kept.p, nptr.p, m + 1);
    const int64_t nn = d2h_scalar(c, nptr.p + m);
    int32_t* ni = dalloc<int32_t>(c, (size_t)nn);
    V* nv = dalloc<V>(c, (size_t)nn);
    drop_zero_entries_kernel<SR><<<grid_for(c, m, 8), 256, 0, c->stream>>>(
        m, out->ptr, out->idx, static_cast<const V*>(out->vals), nptr.p, ni, nv);
    SPG_LAUNCH_CHECK();
    c->launches += 2;
    dfree(c, out->idx);
    dfree(c, out->vals);
    dfree(c, out->ptr);
    out->ptr = nptr.release();
    out->idx = ni;
    out->vals = nv;
    out->nnz = nn;
  }
  if (st) {
    tm.mark(3);
    st->products = products;
    st->nnz_out = out->nnz;
    for (int b = 0; b < kNumBins; ++b) st->rows_per_bin[b] = (int64_t)hcounts[b];
    st->ms_numeric = ms_sym + ms_num;
    st->ms_compact = 0.0;
    st->ms_symbolic = ms_sym;
    st->ms_fold = ms_num;
    st->bitmap_bytes = (int64_t)bm_bytes;
    st->fold_items = nitems;
    st->ms_total = tm.between(0, 3);
    st->ms_analyse = st->ms_total - st->ms_numeric;
    st->kernels = (int64_t)(c->launches - launches0);
    st->output_mode = 3;
  }
  return true;
}

// ---------------------------------------------------------------------------
// Pattern-only semirings (Boolean; semiring.cuh is_pattern_only): rows with
// F > 2048 products get their columns from br_pattern_kernel (count pass,
// rowptr scan, emit pass — any output width, column super-panels of up to
// 2^19 columns, no stored bitmaps, values one()); shorter rows run the ESC /
// hash kernels into U-slot scratch.  Not taken when an operand stores an
// explicit zero() (its products must vanish): run_rows_br / run_rows then.
// ---------------------------------------------------------------------------
template <class SR>
bool run_rows_pattern(spg_ctx* c, const MulSource<SR>& src, const spg_dcsr* r, int64_t ncols_out, spg_dcsr* out,
                      spg_mult_stats* st) {
  using V = typename SR::value_type;
  using Src = MulSource<SR>;
  if constexpr (!is_pattern_only<SR>::value) {
    return false;
  } else {
    static const int on = [] {
      const char* e = std::getenv("SPG_PATTERN");
      return e ? std::atoi(e) : 1;
    }();
    const int64_t m = src.nrows;
    if (!on || c->pipeline != SPG_PIPE_AUTO || m == 0 || ncols_out <= 0 || r->nnz >= (int64_t{1} << 31) - 64)
      return false;
    // explicit zeros in either operand would have to vanish from C: not this path
    {
      int64_t lnnz = 0;
      SPG_CUDA(cudaMemcpyAsync(&lnnz, src.lptr + m, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
      SPG_CUDA(cudaStreamSynchronize(c->stream));
      DBuf<unsigned long long> z(c, 1);
      SPG_CUDA(cudaMemsetAsync(z.p, 0, sizeof(unsigned long long), c->stream));
      if (lnnz > 0) {
        count_zero_values_kernel<SR><<<grid_for(c, lnnz, 256, 8), 256, 0, c->stream>>>(lnnz, src.lval, z.p);
        SPG_LAUNCH_CHECK();
      }
      if (r->nnz > 0) {
        count_zero_values_kernel<SR><<<grid_for(c, r->nnz, 256, 8), 256, 0, c->stream>>>(r->nnz, src.rval, z.p);
        SPG_LAUNCH_CHECK();
      }
      c->launches += 2;
      if (d2h_scalar(c, z.p) != 0) return false;
    }
    NvtxRange nv_all("spg:local_multiply (pattern)");
    PhaseTimer tm(c, st != nullptr);
    const uint64_t launches0 = c->launches;
    tm.mark(0);
    DBuf<int64_t> prods(c, m), ub(c, m + 1), off(c, m + 1), rownnz(c, m + 1);
    DBuf<uint8_t> bins(c, m);
    DBuf<int32_t> colmin(c, 1);
    constexpr int64_t kLongF = 2048;
    analyse_rows_kernel<SR, Src><<<grid_for(c, m, 8), 256, 0, c->stream>>>(
        src, ncols_out, INT64_MAX, 0, 0, 0, 0, 0, kLongF, colmin.p, prods.p, ub.p, bins.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
    SPG_CUDA(cudaMemsetAsync(ub.p + m, 0, sizeof(int64_t), c->stream));
    SPG_CUDA(cudaMemsetAsync(rownnz.p + m, 0, sizeof(int64_t), c->stream));
    exclusive_scan(c, ub.p, off.p, m + 1);
    DBuf<unsigned long long> counts(c, kNumBins + 1);
    SPG_CUDA(cudaMemsetAsync(counts.p, 0, sizeof(unsigned long long) * (kNumBins + 1), c->stream));
    bin_count_kernel<<<grid_for(c, m, 1024, 2), 1024, 0, c->stream>>>(bins.p, m, counts.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
    unsigned long long hcounts[kNumBins];
    int64_t scratch_total = 0;
    SPG_CUDA(cudaMemcpyAsync(hcounts, counts.p, sizeof(hcounts), cudaMemcpyDeviceToHost, c->stream));
    SPG_CUDA(cudaMemcpyAsync(&scratch_total, off.p + m, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    SPG_CUDA(cudaStreamSynchronize(c->stream));
    const int64_t nb = (int64_t)hcounts[kBinBitmap];
    size_t budget = c->scratch_budget;
    if (budget == 0) budget = (size_t)(mem_available(c) * 0.45);
    if ((size_t)scratch_total * (sizeof(int32_t) + sizeof(V)) > budget) return false;
    DBuf<int32_t> sc_cols(c, (size_t)scratch_total + 16);
    DBuf<V> sc_vals(c, (size_t)scratch_total + 16);
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
    int end_bit = 0;
    while ((int64_t{1} << end_bit) < ncols_out) ++end_bit;
    DBuf<int64_t> lists(c, m);
    DBuf<unsigned long long> cursor(c, kNumBins);
    unsigned long long base[kNumBins];
    {
      unsigned long long acc = 0;
      for (int b = 0; b < kNumBins; ++b) {
        base[b] = acc;
        if (b > 0) acc += hcounts[b];
      }
    }
    SPG_CUDA(cudaMemcpyAsync(cursor.p, base, sizeof(base), cudaMemcpyHostToDevice, c->stream));
    bin_scatter_kernel<<<grid_for(c, m, 1024, 2), 1024, 0, c->stream>>>(bins.p, m, cursor.p, lists.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
    const int64_t* brows = lists.p + base[kBinBitmap];
    DBuf<int64_t> bsorted, bk1, bk2;
    if (nb > 1) {
      bk1 = DBuf<int64_t>(c, nb);
      bk2 = DBuf<int64_t>(c, nb);
      bsorted = DBuf<int64_t>(c, nb);
      gather_keys_kernel<<<grid_for(c, nb, 256, 4), 256, 0, c->stream>>>(brows, nb, prods.p, bk1.p);
      SPG_LAUNCH_CHECK();
      ++c->launches;
      size_t bytes = 0;
      SPG_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, bk1.p, bk2.p, brows, bsorted.p, (int)nb, 0,
                                                          64, c->stream));
      ensure_cub_tmp(c, bytes);
      SPG_CUDA(cub::DeviceRadixSort::SortPairsDescending(c->cub_tmp, bytes, bk1.p, bk2.p, brows, bsorted.p, (int)nb,
                                                          0, 64, c->stream));
      ++c->launches;
      brows = bsorted.p;
    }
    if (hcounts[kBinEmpty] > 0) {
      zero_empty_rows_kernel<<<grid_for(c, m, 256, 4), 256, 0, c->stream>>>(bins.p, m, rownnz.p);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    // column super-panels: a 64 KB bitmap (<= 2^19 columns) per pass
    const int spw = std::min(br_words(ncols_out), 16384);
    const int64_t spc = (int64_t)spw * 32;
    const int nsp = (int)((ncols_out + spc - 1) / spc);
    DBuf<int32_t> poff;
    if (nb > 0 && nsp > 1) {
      poff = DBuf<int32_t>(c, (size_t)r->nrows * (nsp + 1));
      panel_offsets_kernel<<<grid_for(c, r->nrows, 8), 256, 0, c->stream>>>(r->nrows, r->ptr, r->idx, nsp, (int)spc,
                                                                            poff.p);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    DBuf<unsigned long long> work(c, 2);
    SPG_CUDA(cudaMemsetAsync(work.p, 0, 2 * sizeof(unsigned long long), c->stream));
    constexpr int kPT = 512;
    const size_t psmem = sizeof(uint32_t) * ((size_t)spw + spw / 32) + BrSegs<V>::bytes(kPT) + 64;
    tm.mark(1);
    {  // count pass (long rows) || short rows into their slots
      NvtxRange nv("spg:pattern count + short rows");
      StreamFork fk(c, 3);
      if (nb > 0) {
        auto kern = br_pattern_kernel<SR, Src, kPT, 0>;
        set_smem(kern, psmem);
        kern<<<resident_grid(c, kern, kPT, psmem, nb), kPT, psmem, fk[0]>>>(src, brows, nb, spw, nsp, poff.p, work.p,
                                                                            rownnz.p, nullptr, nullptr, nullptr);
        SPG_LAUNCH_CHECK();
        ++c->launches;
      }
      RowOut<V> o;
      o.cols = sc_cols.p;
      o.vals = sc_vals.p;
      o.off = off.p;
      o.rownnz = rownnz.p;
      const int64_t* lb = lists.p;
      if (hcounts[kBinHash8K] > 0)
        launch_hash<SR, Src, 8192, 512>(c, fk[1], src, lb + base[kBinHash8K], hcounts[kBinHash8K], 256, end_bit, o);
      if (hcounts[kBinHash4K] > 0)
        launch_hash<SR, Src, 4096, 256>(c, fk[1], src, lb + base[kBinHash4K], hcounts[kBinHash4K], 256, end_bit, o);
      if (hcounts[kBinHash2K] > 0)
        launch_hash<SR, Src, 2048, 128>(c, fk[2], src, lb + base[kBinHash2K], hcounts[kBinHash2K], 256, end_bit, o);
      if (hcounts[kBinEsc512] > 0)
        launch_esc<SR, Src, 128, 4>(c, fk[2], src, lb + base[kBinEsc512], hcounts[kBinEsc512], end_bit, o);
      if (hcounts[kBinWarpEsc] > 0) {
        esc_warp_kernel<SR, Src><<<grid_for(c, hcounts[kBinWarpEsc], 8), 256, 0, fk[2]>>>(
            src, lb + base[kBinWarpEsc], hcounts[kBinWarpEsc], o);
        SPG_LAUNCH_CHECK();
        ++c->launches;
      }
      for (int b : {(int)kBinDense, (int)kBinHashMax, (int)kBinBitRank, (int)kBinRankPanels})
        if (hcounts[b] > 0) fail(SPG_ERR_INTERNAL, "pattern driver: unexpected bin");
      fk.join();
    }
    out->ptr = dalloc<int64_t>(c, m + 1);
    exclusive_scan(c, rownnz.p, out->ptr, m + 1);
    const int64_t nnz = d2h_scalar(c, out->ptr + m);
    tm.mark(2);
    const float ms_cnt = tm.between(1, 2);
    out->nrows = m;
    out->ncols = ncols_out;
    out->nnz = nnz;
    out->idx = dalloc<int32_t>(c, (size_t)nnz);
    out->vals = dalloc<V>(c, (size_t)nnz);
    {  // emit pass (long rows, straight into C) || compaction of the short rows
      NvtxRange nv("spg:pattern emit + short-row compaction");
      StreamFork fk(c, 2);
      if (nb > 0) {
        auto kern = br_pattern_kernel<SR, Src, kPT, 1>;
        set_smem(kern, psmem);
        kern<<<resident_grid(c, kern, kPT, psmem, nb), kPT, psmem, fk[0]>>>(
            src, brows, nb, spw, nsp, poff.p, work.p + 1, nullptr, out->ptr, out->idx, static_cast<V*>(out->vals));
        SPG_LAUNCH_CHECK();
        ++c->launches;
      }
      if (scratch_total > 0) {
        compact_rows_kernel<V><<<grid_for(c, m, 8), 256, 0, fk[1]>>>(m, bins.p, off.p, out->ptr, sc_cols.p,
                                                                   sc_vals.p, out->idx, static_cast<V*>(out->vals));
        SPG_LAUNCH_CHECK();
        ++c->launches;
      }
      fk.join();
    }
    tm.mark(3);
    if (st) {
      const float ms_emit = tm.between(2, 3);
      st->products = products;
      st->nnz_out = out->nnz;
      for (int b = 0; b < kNumBins; ++b) st->rows_per_bin[b] = (int64_t)hcounts[b];
      st->ms_numeric = ms_cnt + ms_emit;
      st->ms_compact = 0.0;
      st->ms_total = tm.between(0, 3);
      st->ms_analyse = st->ms_total - st->ms_numeric;
      st->kernels = (int64_t)(c->launches - launches0);
      st->output_mode = 4;
      st->ms_symbolic = ms_cnt;
      st->ms_fold = ms_emit;
      st->bitmap_bytes = 0;
      st->fold_items = nb;
    }
    return true;
  }
}

}  // namespace spg
