// Width-generic layout kernels (see layout.cuh).
#include <cub/device/device_scan.cuh>

#include <algorithm>

#include "layout.cuh"

namespace spg {

namespace {

__global__ void narrow_kernel(const int64_t* __restrict__ in, int32_t* __restrict__ out, int64_t n,
                              int64_t bound, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = in[i];
    if (v < 0 || v >= bound) *bad = 1;
    out[i] = (int32_t)v;
  }
}

__global__ void widen_kernel(const int32_t* __restrict__ in, int64_t* __restrict__ out, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

__global__ void rebase_rowptr_kernel(const int64_t* __restrict__ in, int64_t* __restrict__ out, int64_t n1) {
  const int64_t base = in[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n1;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i] - base;
}

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* a, int64_t lo, int64_t hi, int64_t x) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void col_count_kernel(int64_t nrows, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                 int64_t b, int64_t e, int64_t* __restrict__ cnt) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < nrows;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t lo = ptr[r], hi = ptr[r + 1];
    const int64_t f = lower_bound_i32(idx, lo, hi, b);
    const int64_t t = lower_bound_i32(idx, f, hi, e);
    cnt[r] = t - f;
  }
}

template <class T>
__global__ void col_fill_kernel(int64_t nrows, const int64_t* __restrict__ ptr, const int32_t* __restrict__ idx,
                                const T* __restrict__ vals, int64_t b, int64_t e,
                                const int64_t* __restrict__ optr, int32_t* __restrict__ oidx,
                                T* __restrict__ ovals) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < nrows; r += nwarps) {
    const int64_t o = optr[r], n = optr[r + 1] - o;
    if (n == 0) continue;
    const int64_t f = lower_bound_i32(idx, ptr[r], ptr[r + 1], b);
    for (int64_t k = lane; k < n; k += 32) {
      oidx[o + k] = (int32_t)(idx[f + k] - b);
      ovals[o + k] = vals[f + k];
    }
  }
}

__global__ void dcsc_scatter_kernel(int64_t njc, const int64_t* __restrict__ jc, const int64_t* __restrict__ cp,
                                    int64_t* __restrict__ lens) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < njc;
       i += (int64_t)gridDim.x * blockDim.x)
    lens[jc[i]] = cp[i + 1] - cp[i];
}

constexpr int kMaxConcat = 64;
struct ConcatParts {
  const int64_t* ptr[kMaxConcat];
  const int32_t* idx[kMaxConcat];
  const void* val[kMaxConcat];
  int64_t shift[kMaxConcat];
};

__global__ void concat_len_kernel(ConcatParts P, int K, int64_t nrows, int64_t* __restrict__ len) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nrows; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t l = 0;
    for (int p = 0; p < K; ++p) l += P.ptr[p][i + 1] - P.ptr[p][i];
    len[i] = l;
  }
}

template <class T>
__global__ void concat_fill_kernel(ConcatParts P, int K, int64_t nrows, const int64_t* __restrict__ optr,
                                   int32_t* __restrict__ oidx, T* __restrict__ oval) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nrows; i += nwarps) {
    int64_t o = optr[i];
    for (int p = 0; p < K; ++p) {
      const int64_t b = P.ptr[p][i], n = P.ptr[p][i + 1] - b;
      const int32_t sh = (int32_t)P.shift[p];
      const int32_t* ix = P.idx[p];
      const T* vv = static_cast<const T*>(P.val[p]);
      for (int64_t k = lane; k < n; k += 32) {
        oidx[o + k] = ix[b + k] + sh;
        oval[o + k] = vv[b + k];
      }
      o += n;
    }
  }
}

__global__ void add_offset_kernel(const int64_t* __restrict__ in, int64_t* __restrict__ out, int64_t n, int64_t add) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i] + add;
}

int blocks_for(spg_ctx* c, int64_t n, int threads = 256) {
  const int64_t want = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)c->sm_count * 16));
}

}  // namespace

// products of every row of L (x) R: F_i = sum over L's entries (i, k) of nnz(R row k)
__global__ void row_products_kernel(int64_t nrows, const int64_t* __restrict__ lptr, const int32_t* __restrict__ lidx,
                                    const int64_t* __restrict__ rptr, int64_t* __restrict__ f) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = warp; i < nrows; i += nwarps) {
    int64_t acc = 0;
    for (int64_t s = lptr[i] + lane; s < lptr[i + 1]; s += 32) {
      const int32_t k = lidx[s];
      acc += rptr[k + 1] - rptr[k];
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) f[i] = acc;
  }
}

void row_products(spg_ctx* c, const spg_dcsr& l, const spg_dcsr& r, int64_t* f) {
  if (l.nrows <= 0) return;
  const int grid = (int)std::min<int64_t>((l.nrows + 7) / 8, (int64_t)c->sm_count * 16);
  row_products_kernel<<<grid, 256, 0, c->stream>>>(l.nrows, l.ptr, l.idx, r.ptr, f);
  SPG_LAUNCH_CHECK();
  ++c->launches;
}

void exclusive_scan_i64(spg_ctx* c, const int64_t* in, int64_t* out, int64_t n) {
  size_t bytes = 0;
  SPG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, c->stream));
  ensure_cub_tmp(c, bytes);
  SPG_CUDA(cub::DeviceScan::ExclusiveSum(c->cub_tmp, bytes, in, out, n, c->stream));
  ++c->launches;
}

void inclusive_scan_i64(spg_ctx* c, const int64_t* in, int64_t* out, int64_t n) {
  size_t bytes = 0;
  SPG_CUDA(cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, n, c->stream));
  ensure_cub_tmp(c, bytes);
  SPG_CUDA(cub::DeviceScan::InclusiveSum(c->cub_tmp, bytes, in, out, n, c->stream));
  ++c->launches;
}

void concat_cols(spg_ctx* c, int K, const spg_dcsr* parts, const int64_t* col_shift, int vs, spg_dcsr* out) {
  if (K < 1 || K > kMaxConcat) fail(SPG_ERR_ARG, "concat: bad part count");
  const int64_t nrows = parts[0].nrows;
  ConcatParts P{};
  int64_t nnz = 0, ncols = 0;
  for (int p = 0; p < K; ++p) {
    if (parts[p].nrows != nrows) fail(SPG_ERR_INTERNAL, "concat_cols: row counts differ");
    P.ptr[p] = parts[p].ptr;
    P.idx[p] = parts[p].idx;
    P.val[p] = parts[p].vals;
    P.shift[p] = col_shift[p];
    nnz += parts[p].nnz;
    ncols = std::max(ncols, col_shift[p] + parts[p].ncols);
  }
  out->nrows = nrows;
  out->ncols = ncols;
  out->nnz = nnz;
  out->ptr = dalloc<int64_t>(c, nrows + 1);
  out->idx = dalloc<int32_t>(c, nnz);
  out->vals = dalloc<char>(c, (size_t)vs * nnz);
  DBuf<int64_t> len(c, nrows + 1);
  SPG_CUDA(cudaMemsetAsync(len.p + nrows, 0, sizeof(int64_t), c->stream));
  if (nrows > 0) {
    concat_len_kernel<<<blocks_for(c, nrows), 256, 0, c->stream>>>(P, K, nrows, len.p);
    SPG_LAUNCH_CHECK();
    ++c->launches;
  }
  exclusive_scan_i64(c, len.p, out->ptr, nrows + 1);
  if (nnz > 0) {
    with_vs(vs, [&](auto tag) {
      using T = typename decltype(tag)::T;
      concat_fill_kernel<T><<<blocks_for(c, nrows * 32), 256, 0, c->stream>>>(P, K, nrows, out->ptr, out->idx,
                                                                             static_cast<T*>(out->vals));
      SPG_LAUNCH_CHECK();
      ++c->launches;
    });
  }
}

void concat_rows(spg_ctx* c, int K, const spg_dcsr* parts, int64_t ncols, int vs, spg_dcsr* out) {
  int64_t nrows = 0, nnz = 0;
  for (int p = 0; p < K; ++p) {
    nrows += parts[p].nrows;
    nnz += parts[p].nnz;
  }
  out->nrows = nrows;
  out->ncols = ncols;
  out->nnz = nnz;
  out->ptr = dalloc<int64_t>(c, nrows + 1);
  out->idx = dalloc<int32_t>(c, nnz);
  out->vals = dalloc<char>(c, (size_t)vs * nnz);
  int64_t r = 0, z = 0;
  for (int p = 0; p < K; ++p) {
    const spg_dcsr& m = parts[p];
    if (m.nrows > 0) {
      add_offset_kernel<<<blocks_for(c, m.nrows), 256, 0, c->stream>>>(m.ptr, out->ptr + r, m.nrows, z);
      SPG_LAUNCH_CHECK();
      ++c->launches;
    }
    if (m.nnz > 0) {
      SPG_CUDA(cudaMemcpyAsync(out->idx + z, m.idx, sizeof(int32_t) * m.nnz, cudaMemcpyDeviceToDevice, c->stream));
      SPG_CUDA(cudaMemcpyAsync(static_cast<char*>(out->vals) + (size_t)vs * z, m.vals, (size_t)vs * m.nnz,
                               cudaMemcpyDeviceToDevice, c->stream));
    }
    r += m.nrows;
    z += m.nnz;
  }
  SPG_CUDA(cudaMemcpyAsync(out->ptr + nrows, &nnz, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
  SPG_CUDA(cudaStreamSynchronize(c->stream));  // &nnz is a host stack value
}

void narrow_indices(spg_ctx* c, const int64_t* in, int32_t* out, int64_t n, int64_t bound) {
  if (n == 0) return;
  DBuf<int> bad(c, 1);
  SPG_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c->stream));
  narrow_kernel<<<blocks_for(c, n), 256, 0, c->stream>>>(in, out, n, bound, bad.p);
  SPG_LAUNCH_CHECK();
  ++c->launches;
  if (d2h_scalar(c, bad.p))
    fail(SPG_ERR_MALFORMED, "index outside [0, " + std::to_string(bound) + ")");
}

void widen_indices(spg_ctx* c, const int32_t* in, int64_t* out, int64_t n) {
  if (n == 0) return;
  widen_kernel<<<blocks_for(c, n), 256, 0, c->stream>>>(in, out, n);
  SPG_LAUNCH_CHECK();
  ++c->launches;
}

void slice_rows_into(spg_ctx* c, const spg_dcsr& m, int64_t b, int64_t e, int vs, const spg_dcsr& out) {
  rebase_rowptr_kernel<<<blocks_for(c, e - b + 1), 256, 0, c->stream>>>(m.ptr + b, out.ptr, e - b + 1);
  SPG_LAUNCH_CHECK();
  ++c->launches;
  if (out.nnz > 0) {
    int64_t lo = 0;
    SPG_CUDA(cudaMemcpyAsync(&lo, m.ptr + b, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    SPG_CUDA(cudaStreamSynchronize(c->stream));
    SPG_CUDA(cudaMemcpyAsync(out.idx, m.idx + lo, sizeof(int32_t) * out.nnz, cudaMemcpyDeviceToDevice, c->stream));
    SPG_CUDA(cudaMemcpyAsync(out.vals, static_cast<const char*>(m.vals) + (size_t)vs * lo,
                             (size_t)vs * out.nnz, cudaMemcpyDeviceToDevice, c->stream));
  }
}

void slice_cols_count(spg_ctx* c, const spg_dcsr& m, int64_t b, int64_t e, int64_t* cnt) {
  SPG_CUDA(cudaMemsetAsync(cnt + m.nrows, 0, sizeof(int64_t), c->stream));
  if (m.nrows == 0) return;
  col_count_kernel<<<blocks_for(c, m.nrows), 256, 0, c->stream>>>(m.nrows, m.ptr, m.idx, b, e, cnt);
  SPG_LAUNCH_CHECK();
  ++c->launches;
}

void slice_cols_fill(spg_ctx* c, const spg_dcsr& m, int64_t b, int64_t e, int vs, const spg_dcsr& out) {
  if (out.nnz == 0 || m.nrows == 0) return;
  with_vs(vs, [&](auto tag) {
    using T = typename decltype(tag)::T;
    col_fill_kernel<T><<<blocks_for(c, m.nrows * 32), 256, 0, c->stream>>>(
        m.nrows, m.ptr, m.idx, static_cast<const T*>(m.vals), b, e, out.ptr, out.idx, static_cast<T*>(out.vals));
    SPG_LAUNCH_CHECK();
    ++c->launches;
  });
}

void dcsc_colptr(spg_ctx* c, int64_t ncols, int64_t njc, const int64_t* jc, const int64_t* cp,
                 int64_t* colptr) {
  DBuf<int64_t> lens(c, ncols + 1);
  SPG_CUDA(cudaMemsetAsync(lens.p, 0, sizeof(int64_t) * (ncols + 1), c->stream));
  if (njc > 0) {
    // lens[c + 1] = run length of column c
    dcsc_scatter_kernel<<<blocks_for(c, njc), 256, 0, c->stream>>>(njc, jc, cp, lens.p + 1);
    SPG_LAUNCH_CHECK();
    ++c->launches;
  }
  inclusive_scan_i64(c, lens.p, colptr, ncols + 1);
}

}  // namespace spg
