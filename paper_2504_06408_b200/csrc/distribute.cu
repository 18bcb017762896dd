// distribute (dist_matrix.hpp:69-111) with the per-block coo_to_csc
// (formats.hpp:138-180) as one device pass over the uploaded COO:
//
//   route   one key per tuple: rank | local column | local row (bit fields
//           sized from the largest block), owner = block_index_of
//           (dist_matrix.hpp:31-37); tuples of other ranks get a sentinel
//           key when one rank's block is wanted
//   sort    one stable LSD radix sort of (key, input position): blocks in
//           rank order, each column-major, duplicates in input order — the
//           reference's stable_sort per piece
//   fold    runs of equal keys fold left to right with SR::add and results
//           equal to SR::is_zero are dropped (SrOps::fold_runs)
//   blocks  colptr by a binary search per column, row ids from the keys,
//           DCSC (jc, cp) by a scan over populated columns when fewer than
//           half are populated (dist_matrix.hpp:97-108)
//
// The keys never leave the device; each block comes back to the host once.
#include <cub/cub.cuh>

#include "instantiate.cuh"
#include "layout.cuh"

namespace spg {
namespace {

SPG_HD int owner_block(int64_t n, int q, int64_t i) {  // dist_matrix.hpp:31-37
  const int64_t base = n / q, extra = n % q, wide = extra * (base + 1);
  return i < wide ? (int)(i / (base + 1)) : (int)(extra + (i - wide) / base);
}

SPG_HD int64_t block_begin(int64_t n, int q, int idx) {  // dist_matrix.hpp:23-28
  const int64_t base = n / q, extra = n % q;
  return idx * base + (idx < extra ? idx : extra);
}

int bits_for(uint64_t max_value) { return max_value == 0 ? 0 : 64 - __builtin_clzll(max_value); }

struct RouteArgs {
  int64_t nrows, ncols;
  int pr, pc, only_rank, rb, cb;
  uint64_t sentinel;
};

__global__ void __launch_bounds__(256) route_kernel(int64_t n, const int64_t* __restrict__ rows,
                                                    const int64_t* __restrict__ cols, RouteArgs a,
                                                    uint64_t* __restrict__ keys, int64_t* __restrict__ order,
                                                    unsigned long long* nvalid, int* bad) {
  unsigned long long mine = 0;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows[k], c = cols[k];
    uint64_t key = a.sentinel;
    if (r < 0 || r >= a.nrows || c < 0 || c >= a.ncols) {
      atomicExch(bad, 1);
    } else {
      const int bi = owner_block(a.nrows, a.pr, r), bj = owner_block(a.ncols, a.pc, c);
      const int rank = bi * a.pc + bj;
      const uint64_t local = ((uint64_t)(c - block_begin(a.ncols, a.pc, bj)) << a.rb) |
                             (uint64_t)(r - block_begin(a.nrows, a.pr, bi));
      if (a.only_rank < 0) {
        key = ((uint64_t)rank << (a.rb + a.cb)) | local;
        ++mine;
      } else if (rank == a.only_rank) {
        key = local;
        ++mine;
      }
    }
    keys[k] = key;
    order[k] = k;
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(nvalid, mine);
}

__global__ void head_flags_kernel(int64_t n, const uint64_t* __restrict__ k, int64_t* __restrict__ f) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    f[p] = p == 0 || k[p] != k[p - 1];
}

__global__ void scatter_heads_kernel(int64_t n, const int64_t* __restrict__ f, const int64_t* __restrict__ pos,
                                     const uint64_t* __restrict__ k, int64_t* __restrict__ heads,
                                     uint64_t* __restrict__ ukeys) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
    if (f[p]) {
      heads[pos[p]] = p;
      ukeys[pos[p]] = k[p];
    }
}

__global__ void keep_flags_kernel(int64_t n, const uint8_t* __restrict__ keep, int64_t* __restrict__ f) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
    f[u] = keep[u] != 0;
}

template <class VT>
__global__ void compact_kept_kernel(int64_t n, const int64_t* __restrict__ f, const int64_t* __restrict__ pos,
                                    const uint64_t* __restrict__ k, const VT* __restrict__ v,
                                    uint64_t* __restrict__ ko, VT* __restrict__ vo) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x)
    if (f[u]) {
      ko[pos[u]] = k[u];
      vo[pos[u]] = v[u];
    }
}

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t n, uint64_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// bounds[r] = first position of rank r (r = 0..nranks).
__global__ void rank_bounds_kernel(int64_t n, const uint64_t* __restrict__ k, int nranks, int shift,
                                   int64_t* __restrict__ bounds) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r <= nranks) bounds[r] = lower_bound_u64(k, n, (uint64_t)r << shift);
}

// colptr[c] = first entry of column c in the block (c = 0..ncols; the search
// key for c = ncols may carry into the rank field, which still bounds the
// block from above); counts the populated columns and flags them for the
// DCSC scan.
__global__ void __launch_bounds__(256) colptr_kernel(int64_t ncols, const uint64_t* __restrict__ k, int64_t nb,
                                                     uint64_t prefix, int rb, int64_t* __restrict__ colptr,
                                                     int64_t* __restrict__ populated_flag,
                                                     unsigned long long* populated) {
  unsigned long long mine = 0;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= ncols;
       c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = lower_bound_u64(k, nb, prefix + ((uint64_t)c << rb));
    colptr[c] = lo;
    if (c < ncols) {
      const int64_t hi = lower_bound_u64(k, nb, prefix + ((uint64_t)(c + 1) << rb));
      populated_flag[c] = hi > lo;
      mine += hi > lo;
    }
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(populated, mine);
}

__global__ void rowids_kernel(int64_t nb, const uint64_t* __restrict__ k, uint64_t row_mask,
                              int64_t* __restrict__ rowids) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < nb; u += (int64_t)gridDim.x * blockDim.x)
    rowids[u] = (int64_t)(k[u] & row_mask);
}

__global__ void dcsc_kernel(int64_t ncols, const int64_t* __restrict__ colptr, const int64_t* __restrict__ f,
                            const int64_t* __restrict__ pos, int64_t* __restrict__ jc, int64_t* __restrict__ cp) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < ncols; c += (int64_t)gridDim.x * blockDim.x)
    if (f[c]) {
      jc[pos[c]] = c;
      cp[pos[c]] = colptr[c];
    }
}

void* must(void* p) {
  if (!p) fail(SPG_ERR_OOM, "distribute: host allocation failed");
  return p;
}

int grid_n(spg_ctx* c, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)c->sm_count * 8));
}

void d2h(spg_ctx* c, void* dst, const void* src, size_t bytes) {
  if (bytes) SPG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
}

}  // namespace

void distribute_coo(spg_ctx* c, const SrOps* ops, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                    const int64_t* cols, const void* vals, int pr, int pc, int only_rank, spg_block* blocks,
                    void* (*halloc)(size_t)) {
  const int vs = ops->value_size;
  const int nranks = pr * pc;
  const int64_t max_rows = std::max<int64_t>(nrows / pr + (nrows % pr ? 1 : 0), 1);
  const int64_t max_cols = std::max<int64_t>(ncols / pc + (ncols % pc ? 1 : 0), 1);
  const int rb = bits_for((uint64_t)max_rows - 1), cb = bits_for((uint64_t)max_cols - 1);
  const int shift = rb + cb;
  const int total = only_rank < 0 ? shift + bits_for((uint64_t)nranks - 1) : shift + 1;
  if (total > 64) fail(SPG_ERR_INVALID_RANGE, "distribute: block extents exceed one 64-bit sort key");
  if (nnz > INT32_MAX) fail(SPG_ERR_INVALID_RANGE, "distribute: more than 2^31 - 1 tuples in one call");
  const uint64_t sentinel = only_rank < 0 ? 0 : (1ull << shift);

  // ---- route + sort + fold (all blocks at once)
  DBuf<uint64_t> keys2;
  DBuf<char> vals2;
  int64_t n2 = 0;
  if (nnz > 0) {
    DBuf<int64_t> drows(c, nnz), dcols(c, nnz);
    DBuf<char> dvals(c, (size_t)vs * nnz);
    SPG_CUDA(cudaMemcpyAsync(drows.p, rows, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, c->stream));
    SPG_CUDA(cudaMemcpyAsync(dcols.p, cols, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, c->stream));
    SPG_CUDA(cudaMemcpyAsync(dvals.p, vals, (size_t)vs * nnz, cudaMemcpyHostToDevice, c->stream));
    DBuf<uint64_t> keys(c, nnz), skeys(c, nnz);
    DBuf<int64_t> order(c, nnz), sorder(c, nnz);
    DBuf<unsigned long long> nvalid(c, 1);
    DBuf<int> bad(c, 1);
    SPG_CUDA(cudaMemsetAsync(nvalid.p, 0, sizeof(unsigned long long), c->stream));
    SPG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c->stream));
    const RouteArgs ra{nrows, ncols, pr, pc, only_rank, rb, cb, sentinel};
    route_kernel<<<grid_n(c, nnz), 256, 0, c->stream>>>(nnz, drows.p, dcols.p, ra, keys.p, order.p, nvalid.p,
                                                          bad.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
    if (d2h_scalar(c, bad.p)) fail(SPG_ERR_MALFORMED, "coo tuple outside the matrix");
    const int64_t nv = (int64_t)d2h_scalar(c, nvalid.p);
    drows.reset();
    dcols.reset();
    size_t bytes = 0;
    SPG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, skeys.p, order.p, sorder.p, (int)nnz, 0, total,
                                             c->stream));
    ensure_cub_tmp(c, bytes);
    SPG_CUDA(cub::DeviceRadixSort::SortPairs(c->cub_tmp, bytes, keys.p, skeys.p, order.p, sorder.p, (int)nnz, 0,
                                             total, c->stream));
    ++c->launches;
    keys.reset();
    order.reset();
    if (nv > 0) {
      DBuf<int64_t> f(c, nv), pos(c, nv);
      head_flags_kernel<<<grid_n(c, nv), 256, 0, c->stream>>>(nv, skeys.p, f.p);
      SPG_LAUNCH_CHECK();
      exclusive_scan(c, f.p, pos.p, nv);
      const int64_t nu = d2h_scalar(c, pos.p + nv - 1) + d2h_scalar(c, f.p + nv - 1);
      DBuf<int64_t> heads(c, nu);
      DBuf<uint64_t> ukeys(c, nu);
      scatter_heads_kernel<<<grid_n(c, nv), 256, 0, c->stream>>>(nv, f.p, pos.p, skeys.p, heads.p, ukeys.p);
      SPG_LAUNCH_CHECK();
      c->launches += 2;
      DBuf<char> uvals(c, (size_t)vs * nu);
      DBuf<uint8_t> keep(c, nu);
      ops->fold_runs(c, nu, heads.p, nv, sorder.p, dvals.p, uvals.p, keep.p);
      DBuf<int64_t> kf(c, nu), kpos(c, nu);
      keep_flags_kernel<<<grid_n(c, nu), 256, 0, c->stream>>>(nu, keep.p, kf.p);
      SPG_LAUNCH_CHECK();
      exclusive_scan(c, kf.p, kpos.p, nu);
      n2 = d2h_scalar(c, kpos.p + nu - 1) + d2h_scalar(c, kf.p + nu - 1);
      keys2 = DBuf<uint64_t>(c, std::max<int64_t>(n2, 1));
      vals2 = DBuf<char>(c, (size_t)vs * std::max<int64_t>(n2, 1));
      with_vs(vs, [&](auto tag) {
        using VT = typename decltype(tag)::T;
        compact_kept_kernel<VT><<<grid_n(c, nu), 256, 0, c->stream>>>(
            nu, kf.p, kpos.p, ukeys.p, reinterpret_cast<const VT*>(uvals.p), keys2.p,
            reinterpret_cast<VT*>(vals2.p));
      });
      SPG_LAUNCH_CHECK();
      c->launches += 2;
    }
  }

  // ---- block boundaries
  std::vector<int64_t> bounds((size_t)nranks + 1, 0);
  if (n2 > 0) {
    if (only_rank < 0) {
      DBuf<int64_t> db(c, nranks + 1);
      rank_bounds_kernel<<<(nranks + 1 + 127) / 128, 128, 0, c->stream>>>(n2, keys2.p, nranks, shift, db.p);
      SPG_LAUNCH_CHECK();
      ++c->launches;
      d2h(c, bounds.data(), db.p, sizeof(int64_t) * (nranks + 1));
      SPG_CUDA(cudaStreamSynchronize(c->stream));
    } else {
      bounds[1] = n2;
    }
  }

  // ---- per block: CSC or DCSC, then D2H
  const int first = only_rank < 0 ? 0 : only_rank, last = only_rank < 0 ? nranks : only_rank + 1;
  for (int r = first; r < last; ++r) {
    spg_block& out = blocks[only_rank < 0 ? r : 0];
    std::memset(&out, 0, sizeof(out));
    const int bi = r / pc, bj = r % pc;
    out.row_begin = block_begin(nrows, pr, bi);
    out.row_end = block_begin(nrows, pr, bi + 1);
    out.col_begin = block_begin(ncols, pc, bj);
    out.col_end = block_begin(ncols, pc, bj + 1);
    const int64_t br = out.row_end - out.row_begin, bc = out.col_end - out.col_begin;
    const int slot = only_rank < 0 ? r : 0;
    const int64_t bs = bounds[(size_t)slot], nb = bounds[(size_t)slot + 1] - bs;
    const uint64_t prefix = only_rank < 0 ? (uint64_t)r << shift : 0;
    DBuf<int64_t> colptr(c, bc + 1), pflag(c, std::max<int64_t>(bc, 1)), ppos(c, std::max<int64_t>(bc, 1));
    DBuf<unsigned long long> npop(c, 1);
    SPG_CUDA(cudaMemsetAsync(npop.p, 0, sizeof(unsigned long long), c->stream));
    colptr_kernel<<<grid_n(c, bc + 1), 256, 0, c->stream>>>(bc, nb > 0 ? keys2.p + bs : nullptr, nb, prefix, rb,
                                                             colptr.p, pflag.p, npop.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
    const int64_t populated = (int64_t)d2h_scalar(c, npop.p);
    DBuf<int64_t> rowids(c, std::max<int64_t>(nb, 1));
    if (nb > 0) {
      rowids_kernel<<<grid_n(c, nb), 256, 0, c->stream>>>(nb, keys2.p + bs, (1ull << rb) - 1, rowids.p);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    // every host array is owned by `out` as soon as it exists (spg_block_free
    // releases a half-built block when a later step fails)
    out.csc.idx = static_cast<int64_t*>(must(halloc(sizeof(int64_t) * std::max<int64_t>(nb, 1))));
    out.csc.vals = must(halloc((size_t)vs * std::max<int64_t>(nb, 1)));
    d2h(c, out.csc.idx, rowids.p, sizeof(int64_t) * nb);
    if (nb > 0) d2h(c, out.csc.vals, vals2.p + (size_t)vs * bs, (size_t)vs * nb);
    if (2 * populated < bc) {  // dist_matrix.hpp:97-108
      out.is_dcsc = 1;
      out.dcsc = spg_hdcsc{br, bc, nb, populated, nullptr, nullptr, out.csc.idx, out.csc.vals};
      out.csc.idx = nullptr;
      out.csc.vals = nullptr;
      out.dcsc.jc = static_cast<int64_t*>(must(halloc(sizeof(int64_t) * std::max<int64_t>(populated, 1))));
      out.dcsc.cp = static_cast<int64_t*>(must(halloc(sizeof(int64_t) * (populated + 1))));
      if (populated > 0) {
        exclusive_scan(c, pflag.p, ppos.p, bc);
        DBuf<int64_t> djc(c, populated), dcp(c, populated);
        dcsc_kernel<<<grid_n(c, bc), 256, 0, c->stream>>>(bc, colptr.p, pflag.p, ppos.p, djc.p, dcp.p);
        SPG_LAUNCH_CHECK();
        ++c->launches;
        d2h(c, out.dcsc.jc, djc.p, sizeof(int64_t) * populated);
        d2h(c, out.dcsc.cp, dcp.p, sizeof(int64_t) * populated);
        SPG_CUDA(cudaStreamSynchronize(c->stream));  // before djc / dcp go back to the pool
      }
      SPG_CUDA(cudaStreamSynchronize(c->stream));
      out.dcsc.cp[populated] = nb;
    } else {
      out.csc.nrows = br;
      out.csc.ncols = bc;
      out.csc.nnz = nb;
      out.csc.ptr = static_cast<int64_t*>(must(halloc(sizeof(int64_t) * (bc + 1))));
      d2h(c, out.csc.ptr, colptr.p, sizeof(int64_t) * (bc + 1));
      SPG_CUDA(cudaStreamSynchronize(c->stream));
    }
  }
}

}  // namespace spg
