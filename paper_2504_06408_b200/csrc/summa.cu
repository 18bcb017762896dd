// One rank's program of the 2.5D Sparse SUMMA (summa25_multiply,
// /root/reference/proj/include/spsumma/summa.hpp:248-349), on a pr x pc grid
// of B200s, one process per GPU.
//
//   prepare   : host CSC/DCSC blocks -> device CSR of their transposes
//               (prepare_block, summa.hpp:30-53; DCSC decompressed on device)
//   stages    : spg_summa_schedule (= the reference's q stages on a square
//               grid; the common refinement of the inner splits otherwise)
//   per round r, stage s (round-major, summa.hpp:290-291):
//     A panel : owner (i, a_col_block) slices rows [half) of its prepared A
//               straight into a packed wire buffer (K6), size triple over the
//               grid row (host path), payload broadcast if nnz > 0
//     B panel : owner (b_row_block, j) column-slices its prepared B the same
//               way, broadcast over the grid column
//     multiply: C^T partial = panB (x) panA (esc(panB, panA), summa.hpp:312)
//               unless a panel is absent (empty-stage guard, :310-321)
//   merge     : GPU merge of the partials in (stage, round) order into the
//               CSC C block (merge_partials, summa.hpp:122-172)
// The ledger mirrors CostLedger (cost_ledger.hpp:31-56) with measured times.
#include <algorithm>
#include <chrono>
#include <functional>
#include <string>
#include <vector>

#include "comm.h"
#include "instantiate.cuh"
#include "layout.cuh"

namespace spg {
const SrOps* ops_for(int sr);
void prepare_block(spg_ctx* c, int sr, const spg_hcsr* csc, const spg_hdcsc* dcsc, spg_dcsr* out);
void free_dcsr(spg_ctx* c, spg_dcsr* m);
int guarded_summa(spg_ctx* c, spg_comm* comm, const std::function<void()>& f);
}  // namespace spg

namespace spg {
namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

struct Panel {
  DBuf<char> buf;
  spg_dcsr view{};
  uint64_t bytes = 0;
  bool present = false;
};

// csr_row_slice of the prepared block into a packed wire buffer.
void pack_rows(spg_ctx* c, const spg_dcsr& m, int64_t b, int64_t e, int vs, Panel& p) {
  int64_t lo = 0, hi = 0;
  SPG_CUDA(cudaMemcpyAsync(&lo, m.ptr + b, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  SPG_CUDA(cudaMemcpyAsync(&hi, m.ptr + e, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
  SPG_CUDA(cudaStreamSynchronize(c->stream));
  const int64_t rows = e - b, nnz = hi - lo;
  p.bytes = panel_bytes(rows, nnz, vs);
  p.buf = DBuf<char>(c, p.bytes);
  p.view = panel_view(p.buf.p, rows, m.ncols, nnz);
  slice_rows_into(c, m, b, e, vs, p.view);
}

// csr_col_slice of the prepared block into a packed wire buffer.
void pack_cols(spg_ctx* c, const spg_dcsr& m, int64_t b, int64_t e, int vs, Panel& p) {
  DBuf<int64_t> cnt(c, m.nrows + 1), ptr(c, m.nrows + 1);
  slice_cols_count(c, m, b, e, cnt.p);
  exclusive_scan_i64(c, cnt.p, ptr.p, m.nrows + 1);
  const int64_t nnz = d2h_scalar(c, ptr.p + m.nrows);
  p.bytes = panel_bytes(m.nrows, nnz, vs);
  p.buf = DBuf<char>(c, p.bytes);
  p.view = panel_view(p.buf.p, m.nrows, e - b, nnz);
  SPG_CUDA(cudaMemcpyAsync(p.view.ptr, ptr.p, sizeof(int64_t) * (m.nrows + 1), cudaMemcpyDeviceToDevice, c->stream));
  slice_cols_fill(c, m, b, e, vs, p.view);
}

// broadcast_panel (summa.hpp:212-235): size triple always, payload if nnz > 0.
// Root side of broadcast_panel: slice + pack (done for all stages up front in
// fused mode, so its host syncs never wait behind in-flight broadcasts).
void pack_panel(spg_ctx* c, spg_comm* comm, int scope, int root, bool by_rows, const spg_dcsr& prepared, int64_t b,
                int64_t e, int vs, Panel& p) {
  if (comm_scope_index(comm, scope) != root) return;
  if (by_rows) pack_rows(c, prepared, b, e, vs, p);
  else pack_cols(c, prepared, b, e, vs, p);
}

// Size triple + payload of an already packed panel (wait = false: device
// broadcasts stay in flight; the caller drains them once).
void send_panel(spg_ctx* c, spg_comm* comm, int scope, int root, int vs, const spg_summa_opts& o, Panel& p,
                spg_ledger& led, bool wait) {
  const bool me = comm_scope_index(comm, scope) == root;
  int64_t triple[3] = {0, 0, 0};
  if (me) {
    triple[0] = p.view.nrows;
    triple[1] = p.view.ncols;
    triple[2] = p.view.nnz;
  }
  const auto t0 = Clock::now();
  comm_exchange_sizes(comm, scope, root, triple);
  ++led.size_exchanges;
  if (me) ++led.rooted_size_exchanges;
  if (triple[2] == 0) {
    led.ms[1] += ms_since(t0);
    return;  // summa.hpp:226: empty panels are not broadcast
  }
  p.present = true;
  if (!me) {
    p.bytes = panel_bytes(triple[0], triple[2], vs);
    p.buf = DBuf<char>(c, p.bytes);
    p.view = panel_view(p.buf.p, triple[0], triple[1], triple[2]);
  }
  const uint64_t thr = (scope == SPG_SCOPE_COL && o.threshold_col) ? o.threshold_col : o.threshold;
  const int path = comm_bcast(comm, scope, root, p.buf.p, p.bytes, o.comm_mode, thr, c->stream, true, wait);
  if (path == SPG_PATH_HOST) {
    ++led.host_bcasts;
    led.bytes_host_path += p.bytes;
    if (me) ++led.rooted_host_bcasts;
  } else {
    ++led.device_bcasts;
    led.bytes_device_path += p.bytes;
    if (me) ++led.rooted_device_bcasts;
  }
  led.ms[1] += ms_since(t0);
}

void broadcast_panel(spg_ctx* c, spg_comm* comm, int scope, int root, bool by_rows, const spg_dcsr& prepared,
                     int64_t b, int64_t e, int vs, const spg_summa_opts& o, Panel& p, spg_ledger& led) {
  const bool me = comm_scope_index(comm, scope) == root;
  int64_t triple[3] = {0, 0, 0};
  if (me) {
    if (by_rows) pack_rows(c, prepared, b, e, vs, p);
    else pack_cols(c, prepared, b, e, vs, p);
    triple[0] = p.view.nrows;
    triple[1] = p.view.ncols;
    triple[2] = p.view.nnz;
  }
  const auto t0 = Clock::now();
  comm_exchange_sizes(comm, scope, root, triple);
  ++led.size_exchanges;
  if (me) ++led.rooted_size_exchanges;
  if (triple[2] == 0) {
    led.ms[1] += ms_since(t0);
    return;  // summa.hpp:226: empty panels are not broadcast
  }
  p.present = true;
  if (!me) {
    p.bytes = panel_bytes(triple[0], triple[2], vs);
    p.buf = DBuf<char>(c, p.bytes);
    p.view = panel_view(p.buf.p, triple[0], triple[1], triple[2]);
  }
  const uint64_t thr = (scope == SPG_SCOPE_COL && o.threshold_col) ? o.threshold_col : o.threshold;
  const int path = comm_bcast(comm, scope, root, p.buf.p, p.bytes, o.comm_mode, thr, c->stream, true);
  if (path == SPG_PATH_HOST) {
    ++led.host_bcasts;
    led.bytes_host_path += p.bytes;
    if (me) ++led.rooted_host_bcasts;
  } else {
    ++led.device_bcasts;
    led.bytes_device_path += p.bytes;
    if (me) ++led.rooted_device_bcasts;
  }
  led.ms[1] += ms_since(t0);
}

}  // namespace
}  // namespace spg

using namespace spg;

extern "C" int spg_summa25_multiply(spg_comm* comm, spg_ctx* c, int sr, int64_t a_nrows, int64_t a_ncols,
                                    int64_t b_ncols, const spg_hcsr* a_csc, const spg_hdcsc* a_dcsc,
                                    const spg_hcsr* b_csc, const spg_hdcsc* b_dcsc, const spg_summa_opts* opts,
                                    spg_dcsr* c_out, spg_ledger* ledger) {
  return guarded_summa(c, comm, [&] {
    if (!comm || !c || !c_out || !opts || !(a_csc || a_dcsc) || !(b_csc || b_dcsc)) fail(SPG_ERR_ARG, "null argument");
    SPG_CUDA(cudaSetDevice(c->device));
    const SrOps* ops = ops_for(sr);
    if (!ops->commutative)  // summa.hpp:262-266 via prepare_block :32-37
      fail(SPG_ERR_UNSUPPORTED_SEMIRING,
           std::string("semiring '") + ops->name +
               "' has a non-commutative multiplication; the distributed transpose-reinterpretation path "
               "supports commutative semirings only");
    const int vs = ops->value_size;
    if (opts->output == SPG_SUMMA_OUT_CHECKSUM && opts->fuse_stages != 1)
      fail(SPG_ERR_ARG, "summa: output = checksum streams the fused multiply (fuse_stages = 1)");
    if (opts->fuse_stages < 0 || opts->fuse_stages > 2) fail(SPG_ERR_ARG, "summa: fuse_stages must be 0, 1 or 2");
    if (opts->output != SPG_SUMMA_OUT_BLOCK && opts->output != SPG_SUMMA_OUT_CHECKSUM)
      fail(SPG_ERR_ARG, "summa: unknown output mode");
    const int pr = comm_pr(comm), pc = comm_pc(comm), i = comm_grid_row(comm), j = comm_grid_col(comm);
    const int64_t inner = a_ncols;
    int64_t arb, are, acb, ace, brb, bre, bcb, bce;
    spg_block_range(a_nrows, pr, i, &arb, &are);
    spg_block_range(inner, pc, j, &acb, &ace);
    spg_block_range(inner, pr, i, &brb, &bre);
    spg_block_range(b_ncols, pc, j, &bcb, &bce);
    auto dims = [](const spg_hcsr* h, const spg_hdcsc* d, int64_t& r, int64_t& cc) {
      r = d ? d->nrows : h->nrows;
      cc = d ? d->ncols : h->ncols;
    };
    int64_t ar, ac, br, bc;
    dims(a_csc, a_dcsc, ar, ac);
    dims(b_csc, b_dcsc, br, bc);
    if (ar != are - arb || ac != ace - acb || br != bre - brb || bc != bce - bcb)
      fail(SPG_ERR_SHAPE, "local blocks do not match the block distribution of " + std::to_string(a_nrows) + "x" +
                              std::to_string(inner) + " by " + std::to_string(inner) + "x" + std::to_string(b_ncols) +
                              " on a " + std::to_string(pr) + "x" + std::to_string(pc) + " grid");
    spg_ledger led{};
    CommCounters& cc0 = comm_counters(comm);
    const double copy0 = cc0.ms_copy;
    const auto t_start = Clock::now();

    // prepare (summa.hpp:278-287)
    spg_dcsr pa{}, pb_own{};
    // C = A (x) A (the same host block passed twice) is prepared once
    const bool same = (a_csc && b_csc && a_csc->ptr == b_csc->ptr && a_csc->idx == b_csc->idx &&
                       a_csc->vals == b_csc->vals) ||
                      (a_dcsc && b_dcsc && a_dcsc->jc == b_dcsc->jc && a_dcsc->cp == b_dcsc->cp &&
                       a_dcsc->rowids == b_dcsc->rowids && a_dcsc->vals == b_dcsc->vals);
    NvtxRange nv_summa("spg:summa25_multiply");
    {
      NvtxRange nv("spg:summa prepare");
      const auto t0 = Clock::now();
      prepare_block(c, sr, a_csc, a_dcsc, &pa);
      if (!same) prepare_block(c, sr, b_csc, b_dcsc, &pb_own);
      SPG_CUDA(cudaStreamSynchronize(c->stream));
      led.ms[0] += ms_since(t0);
    }
    struct Owned {
      spg_ctx* c;
      spg_dcsr* m;
      ~Owned() { free_dcsr(c, m); }
    } own_a{c, &pa}, own_b{c, &pb_own};
    const spg_dcsr& pb = same ? pa : pb_own;

    std::vector<spg_stage> stages(pr + pc + 2);
    const int ns = spg_summa_schedule(inner, pr, pc, stages.data(), (int)stages.size());
    if (ns < 0) fail(SPG_ERR_GRID, "bad grid");
    stages.resize(ns);
    const int rounds = opts->two_round ? 2 : 1;

    struct Part {
      int stage, round;
      spg_dcsr m;
    };
    std::vector<Part> parts;
    // fused mode: every received panel pair is kept (device memory is ample)
    struct Kept {
      int stage, round;
      Panel a, b;
      int64_t a_rows, b_cols;  // panel dims (also for absent panels, from the size triples)
    };
    std::vector<Kept> kept;
    auto free_parts = [&] {
      for (auto& p : parts) free_dcsr(c, &p.m);
      parts.clear();
    };
    const int64_t block_rows = are - arb, block_cols = bce - bcb;
    try {
      // Fused groups: every panel of a group's rounds this rank roots is packed
      // first, then the size exchanges and broadcasts are issued back to back
      // (device ones stay in flight) and drained once — the per-stage host
      // syncs no longer serialise them.
      auto receive_group = [&](int r_lo, int r_hi) {
        NvtxRange nv("spg:summa panels + broadcasts");
        // Fused: pack every panel this rank roots first, then exchange sizes and
        // issue all broadcasts back to back (device ones stay in flight), then
        // drain once — the per-stage host syncs no longer serialise them.
        struct Pending {
          int s, r;
          int64_t rows;
          Panel a, b;
        };
        std::vector<Pending> pend;
        for (int r = r_lo; r < r_hi; ++r)
          for (int s = 0; s < ns; ++s) {
            const spg_stage& st = stages[s];
            int64_t hb, he;
            spg_round_range(st.hi - st.lo, rounds, r, &hb, &he);
            pend.push_back({s, r, he - hb, Panel{}, Panel{}});
            Pending& q = pend.back();
            pack_panel(c, comm, SPG_SCOPE_ROW, st.a_col_block, true, pa, st.a_off + hb, st.a_off + he, vs, q.a);
            pack_panel(c, comm, SPG_SCOPE_COL, st.b_row_block, false, pb, st.b_off + hb, st.b_off + he, vs, q.b);
          }
        for (auto& q : pend) {
          const spg_stage& st = stages[q.s];
          send_panel(c, comm, SPG_SCOPE_ROW, st.a_col_block, vs, *opts, q.a, led, false);
          send_panel(c, comm, SPG_SCOPE_COL, st.b_row_block, vs, *opts, q.b, led, false);
        }
        {
          const auto t0 = Clock::now();
          comm_bcast_wait(comm, c->stream);
          led.ms[1] += ms_since(t0);
        }
        uint64_t total = 0;
        for (auto& q : pend) {
          total += (q.a.present ? q.a.bytes : 0) + (q.b.present ? q.b.bytes : 0);
          if (!(q.a.present && q.b.present)) ++led.skipped_stages;
          kept.push_back({q.s, q.r, std::move(q.a), std::move(q.b), q.rows, block_cols});
        }
        if (total > led.peak_bcast_buffer_bytes) led.peak_bcast_buffer_bytes = total;
      };
      for (int r = 0; r < (opts->fuse_stages ? 0 : rounds); ++r) {
        for (int s = 0; s < ns; ++s) {
          const spg_stage& st = stages[s];
          int64_t hb, he;
          spg_round_range(st.hi - st.lo, rounds, r, &hb, &he);
          // A panel: rows [a_off + hb, a_off + he) of the prepared A (A's local columns)
          Panel pana, panb;
          broadcast_panel(c, comm, SPG_SCOPE_ROW, st.a_col_block, true, pa, st.a_off + hb, st.a_off + he, vs, *opts,
                          pana, led);
          // B panel: columns [b_off + hb, b_off + he) of the prepared B (B's local rows)
          broadcast_panel(c, comm, SPG_SCOPE_COL, st.b_row_block, false, pb, st.b_off + hb, st.b_off + he, vs,
                          *opts, panb, led);
          if (opts->fuse_stages) {
            const uint64_t resident = (pana.present ? pana.bytes : 0) + (panb.present ? panb.bytes : 0);
            uint64_t total = resident;
            for (auto& k : kept) total += (k.a.present ? k.a.bytes : 0) + (k.b.present ? k.b.bytes : 0);
            if (total > led.peak_bcast_buffer_bytes) led.peak_bcast_buffer_bytes = total;
            if (!(pana.present && panb.present)) ++led.skipped_stages;
            kept.push_back({s, r, std::move(pana), std::move(panb), he - hb, block_cols});
            continue;
          }
          const uint64_t resident = (pana.present ? pana.bytes : 0) + (panb.present ? panb.bytes : 0);
          if (resident > led.peak_bcast_buffer_bytes) led.peak_bcast_buffer_bytes = resident;
          if (pana.present && panb.present) {
            const auto t0 = Clock::now();
            spg_mult_stats ms{};
            spg_dcsr ct{};
            ops->local_multiply(c, &panb.view, &pana.view, &ct, &ms);
            led.ms[2] += ms_since(t0);
            led.products += ms.products;
            ++led.local_multiply_calls;
            parts.push_back({s, r, ct});
          } else {
            ++led.skipped_stages;
          }
        }
      }
      auto multiply_kept = [&]() -> spg_dcsr {
        NvtxRange nv("spg:summa fused multiply");
        // C^T = [panB_0 | panB_1 | ...] (x) [panA_0; panA_1; ...]  in (stage, round) order
        // = ascending inner index k, so the fold order equals the serial reference's.
        const auto t0 = Clock::now();
        std::stable_sort(kept.begin(), kept.end(), [](const Kept& x, const Kept& y) {
          return x.stage != y.stage ? x.stage < y.stage : x.round < y.round;
        });
        std::vector<spg_dcsr> bs, as;
        std::vector<int64_t> shift;
        std::vector<DBuf<int64_t>> empties;  // zero rowptrs for panels that were not broadcast
        int64_t off = 0;
        for (auto& k : kept) {
          auto empty_view = [&](int64_t rows, int64_t cols) {
            empties.emplace_back(c, rows + 1);
            SPG_CUDA(cudaMemsetAsync(empties.back().p, 0, sizeof(int64_t) * (rows + 1), c->stream));
            spg_dcsr v{rows, cols, 0, empties.back().p, nullptr, nullptr};
            return v;
          };
          bs.push_back(k.b.present ? k.b.view : empty_view(block_cols, k.a_rows));
          as.push_back(k.a.present ? k.a.view : empty_view(k.a_rows, block_rows));
          shift.push_back(off);
          off += k.a_rows;
        }
        spg_dcsr L{}, R{};
        if (!kept.empty()) {
          concat_cols(c, (int)bs.size(), bs.data(), shift.data(), vs, &L);
          concat_rows(c, (int)as.size(), as.data(), block_rows, vs, &R);
        }
        kept.clear();  // panel buffers are released (stream-ordered) once copied
        empties.clear();
        struct OwnedLR {
          spg_ctx* c;
          spg_dcsr *l, *r;
          ~OwnedLR() {
            free_dcsr(c, l);
            free_dcsr(c, r);
          }
        } own_lr{c, &L, &R};
        spg_mult_stats ms{};
        spg_dcsr ct{};
        if (L.nrows == 0 && R.nrows == 0) {
          L.nrows = block_cols;
        }
        led.left_nnz = L.nnz;
        if (off == 0) {  // no inner dimension: empty product
          ct.nrows = block_cols;
          ct.ncols = block_rows;
          ct.ptr = dalloc<int64_t>(c, block_cols + 1);
          ct.idx = dalloc<int32_t>(c, 1);
          ct.vals = dalloc<char>(c, vs);
          SPG_CUDA(cudaMemsetAsync(ct.ptr, 0, sizeof(int64_t) * (block_cols + 1), c->stream));
        } else if (opts->output == SPG_SUMMA_OUT_CHECKSUM) {
          // C block larger than HBM: the fused product in column batches of
          // the block (rows of C^T), each checksummed and released
          DBuf<int64_t> f(c, (size_t)L.nrows);
          row_products(c, L, R, f.p);
          std::vector<int64_t> hf((size_t)L.nrows);
          SPG_CUDA(cudaMemcpyAsync(hf.data(), f.p, sizeof(int64_t) * L.nrows, cudaMemcpyDeviceToHost, c->stream));
          SPG_CUDA(cudaStreamSynchronize(c->stream));
          const uint64_t budget0 = opts->batch_bytes ? opts->batch_bytes : (uint64_t)(mem_available(c) * 0.25);
          const uint64_t per = 4 + (uint64_t)vs;  // bytes per C entry
          // equal batches (total / ceil(total / budget)): consecutive batches
          // then need equal buffers, which the block cache hands back instead
          // of growing the pool (a fresh 30 GB block costs up to 1 s to map)
          uint64_t total_b = 0;
          for (int64_t r = 0; r < L.nrows; ++r) total_b += (uint64_t)std::min<int64_t>(hf[r], R.ncols) * per;
          const uint64_t nbat = std::max<uint64_t>(1, (total_b + budget0 - 1) / std::max<uint64_t>(budget0, 1));
          const uint64_t budget = std::min<uint64_t>(budget0, (total_b / nbat) + (total_b / nbat) / 32);  // +3 %: no stub batch
          for (int64_t r0 = 0; r0 < L.nrows;) {
            int64_t r1 = r0;
            uint64_t acc = 0;
            while (r1 < L.nrows) {
              const uint64_t e = (uint64_t)std::min<int64_t>(hf[r1], R.ncols) * per;  // nnz <= min(F, width)
              if (r1 > r0 && acc + e > budget) break;
              acc += e;
              ++r1;
            }
            spg_dcsr lv = L;
            lv.nrows = r1 - r0;
            lv.ptr = L.ptr + r0;
            spg_dcsr cb{};
            spg_mult_stats bs{};
            const auto tb = Clock::now();
            ops->local_multiply(c, &lv, &R, &cb, &bs);
            if (HostTrace::limit_ms() >= 0)
              std::fprintf(stderr, "[spg-host] summa batch rows [%lld, %lld) products %lld nnz %lld mode %lld: %.1f ms "
                                   "(analyse %.1f numeric %.1f compact %.1f) budget %.1f GB, available %.1f GB, "
                                   "cached %.1f GB\n",
                           (long long)r0, (long long)r1, (long long)bs.products, (long long)cb.nnz,
                           (long long)bs.output_mode, ms_since(tb), bs.ms_analyse, bs.ms_numeric, bs.ms_compact,
                           budget / 1e9, mem_available(c) / 1e9, c->big_cached / 1e9);
            spg_dcsr csc = cb;  // CSR of C^T rows [r0, r1) == CSC of C columns bcb + [r0, r1)
            csc.nrows = block_rows;
            csc.ncols = r1 - r0;
            led.checksum_part += ops->checksum_part(c, &csc, 1, arb, bcb + r0);
            led.nnz_out += cb.nnz;
            ms.products += bs.products;
            free_dcsr(c, &cb);
            ++led.batches;
            ++led.local_multiply_calls;
            r0 = r1;
          }
          ct.nrows = block_cols;
          ct.ncols = block_rows;
          ct.ptr = dalloc<int64_t>(c, block_cols + 1);
          ct.idx = dalloc<int32_t>(c, 1);
          ct.vals = dalloc<char>(c, vs);
          SPG_CUDA(cudaMemsetAsync(ct.ptr, 0, sizeof(int64_t) * (block_cols + 1), c->stream));
        } else {
          ops->local_multiply(c, &L, &R, &ct, &ms);
          ++led.local_multiply_calls;
          led.nnz_out = ct.nnz;
          led.batches = 1;
        }
        led.products += ms.products;
        SPG_CUDA(cudaStreamSynchronize(c->stream));
        led.ms[2] += ms_since(t0);
        return ct;
      };
      // fuse_stages 1: one fusion group (all rounds; peak buffer = every
      // panel); 2: one group per round, the round products folded by the GPU
      // merge (merge_partials, summa.hpp:122-172) — the 2.5D memory bound:
      // only one round's panels are resident (SPEC acceptance 9).
      const int groups = opts->fuse_stages == 2 ? rounds : 1;
      if (opts->fuse_stages) {
        for (int g = 0; g < groups; ++g) {
          if (groups == 1) receive_group(0, rounds);
          else receive_group(g, g + 1);
          spg_dcsr ct = multiply_kept();
          if (groups == 1) {
            *c_out = ct;
            c_out->nrows = block_rows;
            c_out->ncols = block_cols;
          } else {
            parts.push_back({0, g, ct});
          }
        }
      }
      if (opts->fuse_stages && groups == 1) {
        // done: c_out holds the fused product
      } else {
        // merge (summa.hpp:325-328), stage-major / round-minor
        const auto t0 = Clock::now();
        std::stable_sort(parts.begin(), parts.end(), [](const Part& x, const Part& y) {
          return x.stage != y.stage ? x.stage < y.stage : x.round < y.round;
        });
        if (parts.empty()) {
          c_out->nrows = block_rows;
          c_out->ncols = block_cols;
          c_out->nnz = 0;
          c_out->ptr = dalloc<int64_t>(c, block_cols + 1);
          c_out->idx = dalloc<int32_t>(c, 1);
          c_out->vals = dalloc<char>(c, vs);
          SPG_CUDA(cudaMemsetAsync(c_out->ptr, 0, sizeof(int64_t) * (block_cols + 1), c->stream));
        } else if (parts.size() == 1) {
          // a single partial already is the CSR of C^T == CSC of C
          *c_out = parts[0].m;
          c_out->nrows = block_rows;
          c_out->ncols = block_cols;
          parts.clear();
        } else {
          std::vector<spg_dcsr> ps;
          for (auto& p : parts) ps.push_back(p.m);
          spg_dcsr out{};
          ops->merge(c, (int)ps.size(), ps.data(), block_cols, block_rows, &out, nullptr);
          out.nrows = block_rows;
          out.ncols = block_cols;
          *c_out = out;
          free_parts();
        }
        SPG_CUDA(cudaStreamSynchronize(c->stream));
        led.ms[3] += ms_since(t0);
        led.nnz_out = c_out->nnz;
        led.batches = 1;
      }
    } catch (...) {
      free_parts();
      throw;
    }
    led.ms[4] = comm_counters(comm).ms_copy - copy0;
    led.ms_total = ms_since(t_start);
    if (ledger) *ledger = led;
  });
}

// ---------------------------------------------------------------------------
// gather (dist_matrix.hpp: gather): every rank's CSC block of C
// to one rank, assembled on that rank's GPU into the full CSC matrix.  Blocks
// travel packed (wire format) over NCCL send/recv; the root merges each
// column's pieces in block-row order (row ranges are disjoint and
// increasing, so no sort is needed).
// ---------------------------------------------------------------------------
namespace spg {
namespace {

constexpr int kMaxGatherParts = 32;
struct GatherParts {
  const int64_t* ptr[kMaxGatherParts];
  const int32_t* idx[kMaxGatherParts];
  const unsigned char* vals[kMaxGatherParts];
  int64_t r0[kMaxGatherParts], c0[kMaxGatherParts], nc[kMaxGatherParts];
  int n;  // parts sorted by (c0, r0)
};

__device__ __forceinline__ void parts_of_col(const GatherParts& g, int64_t c, int& first, int& last) {
  first = last = -1;
  for (int k = 0; k < g.n; ++k)
    if (c >= g.c0[k] && c < g.c0[k] + g.nc[k]) {
      if (first < 0) first = k;
      last = k;
    }
}

__global__ void gather_count_kernel(GatherParts g, int64_t ncols, int64_t* cnt) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncols; c += (int64_t)gridDim.x * blockDim.x) {
    int f, l;
    parts_of_col(g, c, f, l);
    int64_t n = 0;
    for (int k = f; k >= 0 && k <= l; ++k) {
      const int64_t lc = c - g.c0[k];
      n += g.ptr[k][lc + 1] - g.ptr[k][lc];
    }
    cnt[c] = n;
  }
}

__global__ void gather_fill_kernel(GatherParts g, int64_t ncols, int vs, const int64_t* __restrict__ colptr,
                                   int32_t* __restrict__ idx, unsigned char* __restrict__ vals) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = warp; c < ncols; c += nwarps) {
    int f, l;
    parts_of_col(g, c, f, l);
    int64_t d = colptr[c];
    for (int k = f; k >= 0 && k <= l; ++k) {
      const int64_t lc = c - g.c0[k];
      const int64_t b = g.ptr[k][lc], n = g.ptr[k][lc + 1] - b;
      for (int64_t e = lane; e < n; e += 32) {
        idx[d + e] = (int32_t)(g.idx[k][b + e] + g.r0[k]);
        for (int q = 0; q < vs; ++q) vals[(d + e) * vs + q] = g.vals[k][(b + e) * vs + q];
      }
      d += n;
    }
  }
}

}  // namespace
}  // namespace spg

extern "C" int spg_gather(spg_comm* comm, spg_ctx* c, int sr, const spg_dcsr* blk, int64_t row_off, int64_t col_off,
                          int64_t nrows, int64_t ncols, int root, spg_dcsr* out) {
  return guarded_summa(c, comm, [&] {
    if (!comm || !c || !blk || !out) fail(SPG_ERR_ARG, "null argument");
    SPG_CUDA(cudaSetDevice(c->device));
    const int vs = ops_for(sr)->value_size;
    const int world = comm_world_size(comm), me = comm_world_rank(comm);
    if (world > kMaxGatherParts) fail(SPG_ERR_GRID, "gather supports up to 32 ranks");
    // my block, packed (CSC: ptr over its columns)
    const size_t bytes = panel_bytes(blk->ncols, blk->nnz, vs);
    DBuf<char> mine(c, bytes);
    spg_dcsr v = panel_view(mine.p, blk->ncols, blk->nrows, blk->nnz);
    SPG_CUDA(cudaMemcpyAsync(v.ptr, blk->ptr, sizeof(int64_t) * (blk->ncols + 1), cudaMemcpyDeviceToDevice, c->stream));
    if (blk->nnz) {
      SPG_CUDA(cudaMemcpyAsync(v.idx, blk->idx, sizeof(int32_t) * blk->nnz, cudaMemcpyDeviceToDevice, c->stream));
      SPG_CUDA(cudaMemcpyAsync(v.vals, blk->vals, (size_t)vs * blk->nnz, cudaMemcpyDeviceToDevice, c->stream));
    }
    const int64_t meta[6] = {blk->nnz, row_off, col_off, blk->nrows, blk->ncols, (int64_t)bytes};
    std::vector<int64_t> all((size_t)world * 6);
    comm_allgather_i64(comm, meta, 6, all.data(), c->stream);
    std::vector<DBuf<char>> bufs(world);
    std::vector<void*> recv(world, nullptr);
    std::vector<uint64_t> rbytes(world, 0);
    if (me == root)
      for (int r = 0; r < world; ++r) {
        rbytes[r] = (uint64_t)all[r * 6 + 5];
        if (r != root) {
          bufs[r] = DBuf<char>(c, rbytes[r]);
          recv[r] = bufs[r].p;
        } else {
          recv[r] = mine.p;
        }
      }
    comm_gather_bytes(comm, root, mine.p, bytes, recv.data(), rbytes.data(), c->stream);
    out->nrows = nrows;
    out->ncols = ncols;
    out->nnz = 0;
    out->ptr = nullptr;
    out->idx = nullptr;
    out->vals = nullptr;
    if (me != root) return;
    std::vector<int> order(world);
    for (int r = 0; r < world; ++r) order[r] = r;
    std::sort(order.begin(), order.end(), [&](int a, int b) {
      return std::make_pair(all[a * 6 + 2], all[a * 6 + 1]) < std::make_pair(all[b * 6 + 2], all[b * 6 + 1]);
    });
    GatherParts g{};
    g.n = world;
    for (int k = 0; k < world; ++k) {
      const int r = order[k];
      const spg_dcsr pv = panel_view(recv[r], all[r * 6 + 4], all[r * 6 + 3], all[r * 6 + 0]);
      g.ptr[k] = pv.ptr;
      g.idx[k] = pv.idx;
      g.vals[k] = static_cast<const unsigned char*>(pv.vals);
      g.r0[k] = all[r * 6 + 1];
      g.c0[k] = all[r * 6 + 2];
      g.nc[k] = all[r * 6 + 4];
    }
    DBuf<int64_t> cnt(c, ncols + 1);
    SPG_CUDA(cudaMemsetAsync(cnt.p + ncols, 0, sizeof(int64_t), c->stream));
    gather_count_kernel<<<(int)std::min<int64_t>((ncols + 255) / 256, (int64_t)c->sm_count * 16), 256, 0, c->stream>>>(
        g, ncols, cnt.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
    out->ptr = dalloc<int64_t>(c, ncols + 1);
    exclusive_scan_i64(c, cnt.p, out->ptr, ncols + 1);
    out->nnz = d2h_scalar(c, out->ptr + ncols);
    out->idx = dalloc<int32_t>(c, (size_t)std::max<int64_t>(out->nnz, 1));
    out->vals = dalloc<unsigned char>(c, (size_t)vs * std::max<int64_t>(out->nnz, 1));
    gather_fill_kernel<<<(int)std::min<int64_t>((ncols + 7) / 8, (int64_t)c->sm_count * 16), 256, 0, c->stream>>>(
        g, ncols, vs, out->ptr, out->idx, static_cast<unsigned char*>(out->vals));
    SPG_LAUNCH_CHECK();
    ++c->launches;
    SPG_CUDA(cudaStreamSynchronize(c->stream));
  });
}
