// Shared host/device plumbing for the B200 SpGEMM engine: status codes that
// mirror the reference's exception classes (common.hpp:12-73), the per-GPU
// context (device, stream, stream-ordered memory pool) and device buffers.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <utility>

#include "../../include/spgemm_b200.h"

namespace spg {

// A typed error that the C-ABI turns into an SPG_ERR_* status.
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(int status, const std::string& msg) { throw Error(status, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    const int st = (e == cudaErrorMemoryAllocation) ? SPG_ERR_OOM : SPG_ERR_CUDA;
    fail(st, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                 std::to_string(line) + ")");
  }
}
#define SPG_CUDA(x) ::spg::cuda_check((x), #x, __FILE__, __LINE__)
#define SPG_LAUNCH_CHECK() ::spg::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__)

}  // namespace spg

// Per-GPU context.  One host thread (or process) drives one context.
struct spg_ctx {
  int device = 0;
  int sm_count = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaMemPool_t pool = nullptr;
  std::string last_error;
  // cub temporary storage, grown on demand and reused
  void* cub_tmp = nullptr;
  size_t cub_tmp_bytes = 0;
  // per-phase timing of the last local multiply / merge (CUDA events)
  cudaEvent_t ev[8] = {};
  cudaStream_t aux[4] = {};      // side streams for concurrent bins
  cudaEvent_t aux_ev[4] = {};
  cudaEvent_t fork_ev = nullptr;
  uint64_t launches = 0;  // kernels launched by this context (evidence counter)
  size_t scratch_budget = 0;  // bytes the row-batched numeric pass may use (0 = auto)
};

namespace spg {

// Stream-ordered device allocation from the context's pool.
template <class T>
T* dalloc(spg_ctx* c, size_t n) {
  if (n == 0) n = 1;
  void* p = nullptr;
  SPG_CUDA(cudaMallocAsync(&p, n * sizeof(T), c->stream));
  return static_cast<T*>(p);
}
inline void dfree(spg_ctx* c, void* p) {
  if (p) SPG_CUDA(cudaFreeAsync(p, c->stream));
}

// RAII device buffer (freed stream-ordered on the context stream).
template <class T>
struct DBuf {
  spg_ctx* c = nullptr;
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  DBuf(spg_ctx* ctx, size_t count) : c(ctx), p(dalloc<T>(ctx, count)), n(count) {}
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : c(o.c), p(o.p), n(o.n) { o.p = nullptr; }
  DBuf& operator=(DBuf&& o) noexcept {
    reset();
    c = o.c; p = o.p; n = o.n; o.p = nullptr;
    return *this;
  }
  ~DBuf() { reset(); }
  void reset() {
    if (p) cudaFreeAsync(p, c->stream);
    p = nullptr;
  }
  T* release() { T* q = p; p = nullptr; return q; }
};

inline void ensure_cub_tmp(spg_ctx* c, size_t bytes) {
  if (bytes <= c->cub_tmp_bytes) return;
  if (c->cub_tmp) SPG_CUDA(cudaFreeAsync(c->cub_tmp, c->stream));
  c->cub_tmp_bytes = bytes + (bytes >> 2) + 4096;
  SPG_CUDA(cudaMallocAsync(&c->cub_tmp, c->cub_tmp_bytes, c->stream));
}

template <class T>
T d2h_scalar(spg_ctx* c, const T* dptr) {
  T v{};
  SPG_CUDA(cudaMemcpyAsync(&v, dptr, sizeof(T), cudaMemcpyDeviceToHost, c->stream));
  SPG_CUDA(cudaStreamSynchronize(c->stream));
  return v;
}

inline int ceil_div(int64_t a, int64_t b) { return static_cast<int>((a + b - 1) / b); }

}  // namespace spg
