// Shared host/device plumbing for the B200 SpGEMM engine: status codes that
// mirror the reference's exception classes (common.hpp:12-73), the per-GPU
// context (device, stream, stream-ordered memory pool) and device buffers.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <unordered_map>
#include <stdexcept>
#include <string>
#include <utility>

#include <nvtx3/nvToolsExt.h>

#include "../../include/spgemm_b200.h"

namespace spg {

// A typed error that the C-ABI turns into an SPG_ERR_* status (default
// visibility: user semiring libraries throw it across the library boundary).
struct __attribute__((visibility("default"))) Error : std::runtime_error {
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
  cudaMemPool_t pool = nullptr;      // device default pool: small buffers
  cudaMemPool_t big_pool = nullptr;  // private pool for buffers >= kBigAlloc (no fragmentation by small ones)
  // Cache of large device buffers: freed blocks are kept and handed out
  // again (stream-ordered on `stream`) to requests of nearly the same size,
  // so steady-state calls never map fresh memory.
  std::multimap<size_t, void*> big_free;
  std::unordered_map<void*, size_t> big_live;
  size_t big_cached = 0;
  size_t free_snap = 0;              // cudaMemGetInfo free bytes at the last snapshot
  size_t reserved_snap = 0;          // pool bytes reserved at that snapshot
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
  int pipeline = 0;           // SPG_PIPE_AUTO (bitmap-rank when eligible) or SPG_PIPE_BINS
};

namespace spg {

// SPG_HOST_TRACE=<ms>: report host calls that block longer than <ms>
// (stalls there show up as idle gaps inside the device-timed phases).
struct HostTrace {
  const char* what;
  size_t arg;
  std::chrono::steady_clock::time_point t0;
  static double limit_ms() {
    static const double v = [] {
      const char* e = std::getenv("SPG_HOST_TRACE");
      return e ? std::atof(e) : -1.0;
    }();
    return v;
  }
  HostTrace(const char* w, size_t a = 0) : what(w), arg(a), t0(std::chrono::steady_clock::now()) {}
  ~HostTrace() {
    const double lim = limit_ms();
    if (lim < 0) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (ms >= lim) std::fprintf(stderr, "[spg-host] %s (%zu) %.3f ms\n", what, arg, ms);
  }
};

// Device-side bounds checks of the checked build (make variant VNAME=checks
// VFLAGS=-DSPG_CHECKS): a violated invariant traps the kernel (a CUDA error
// on the next sync) instead of reading or writing out of bounds.  Used in
// place of compute-sanitizer, which this GPU pool does not allow.
#ifdef SPG_CHECKS
#define SPG_DCHECK(cond) \
  do {                   \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define SPG_DCHECK(cond)   \
  do {                     \
    (void)sizeof((cond));  \
  } while (0)  // unevaluated: no code, but the operands count as used
#endif

// NVTX range for profilers (nsys / ncu --nvtx): host-side phase markers,
// no cost without an attached tool (NVTX v3, header-only).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Stream-ordered device allocation.  Large buffers come from the context's
// private pool, so the many small per-call buffers never split the big
// cached blocks (a split forces the pool to map fresh memory: tens of ms).
constexpr size_t kBigAlloc = size_t(16) << 20;
inline cudaError_t pool_alloc(spg_ctx* c, void** p, size_t bytes) {
  return (bytes >= kBigAlloc && c->big_pool) ? cudaMallocFromPoolAsync(p, bytes, c->big_pool, c->stream)
                                             : cudaMallocAsync(p, bytes, c->stream);
}
// Returns every cached large block to the pool and the pools' idle reserve
// to the device.
inline void release_cached(spg_ctx* c) {
  HostTrace ht("release_cached (out of memory)", c->big_cached);
  for (auto& kv : c->big_free) cudaFreeAsync(kv.second, c->stream);
  c->big_free.clear();
  c->big_cached = 0;
  SPG_CUDA(cudaStreamSynchronize(c->stream));
  SPG_CUDA(cudaMemPoolTrimTo(c->pool, 0));
  if (c->big_pool) SPG_CUDA(cudaMemPoolTrimTo(c->big_pool, 0));
}
// Allocation; large requests first try the block cache (a cached block of
// size in [need, need * 9/8]).  Out of memory: release the caches, retry
// once; allow_fail then returns nullptr instead of failing.
inline void* dalloc_bytes(spg_ctx* c, size_t bytes, bool allow_fail) {
  void* p = nullptr;
  HostTrace ht("cudaMallocAsync", bytes);
  const bool big = bytes >= kBigAlloc;
  if (big) {
    // size classes: rounded up to 1/16 of the request's power of two (>= 2 MB),
    // so the slightly different buffers of consecutive calls (streamed
    // batches) reuse one cached block instead of growing the pool — a fresh
    // 30 GB block costs 0.2-1.2 s of mapping
    int lg = 63 - __builtin_clzll((unsigned long long)bytes);
    const size_t gran = std::max<size_t>(size_t(2) << 20, size_t(1) << (lg > 4 ? lg - 4 : 0));
    bytes = (bytes + gran - 1) / gran * gran;
    auto it = c->big_free.lower_bound(bytes);
    if (it != c->big_free.end() && it->first <= bytes + bytes / 2) {  // the smallest cached fit, <= 1.5x
      p = it->second;
      c->big_live[p] = it->first;
      c->big_cached -= it->first;
      c->big_free.erase(it);
      return p;
    }
  }
  cudaError_t e = pool_alloc(c, &p, bytes);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    release_cached(c);
    e = pool_alloc(c, &p, bytes);
  }
  if (e == cudaErrorMemoryAllocation && allow_fail) {
    cudaGetLastError();
    return nullptr;
  }
  SPG_CUDA(e);
  if (big) c->big_live[p] = bytes;
  return p;
}
// Stream-ordered free; large blocks go back to the cache.
inline void dfree_bytes(spg_ctx* c, void* p) {
  if (!p) return;
  auto it = c->big_live.find(p);
  if (it != c->big_live.end()) {
    c->big_free.emplace(it->second, p);
    c->big_cached += it->second;
    c->big_live.erase(it);
    return;
  }
  SPG_CUDA(cudaFreeAsync(p, c->stream));
}
template <class T>
T* dalloc(spg_ctx* c, size_t n) {
  return static_cast<T*>(dalloc_bytes(c, std::max<size_t>(n, 1) * sizeof(T), false));
}
// As dalloc, but an out-of-memory result returns nullptr instead of failing.
template <class T>
T* try_dalloc(spg_ctx* c, size_t n) {
  return static_cast<T*>(dalloc_bytes(c, std::max<size_t>(n, 1) * sizeof(T), true));
}

inline size_t pool_attr(cudaMemPool_t p, cudaMemPoolAttr a) {
  uint64_t v = 0;
  if (p) cudaMemPoolGetAttribute(p, a, &v);
  return (size_t)v;
}
// Re-reads free device memory (cudaMemGetInfo can block for tens of ms, so
// it runs at context creation and after an allocation failure only).
inline void mem_snapshot(spg_ctx* c) {
  size_t fr = 0, tot = 0;
  SPG_CUDA(cudaMemGetInfo(&fr, &tot));
  c->free_snap = fr;
  c->reserved_snap = pool_attr(c->pool, cudaMemPoolAttrReservedMemCurrent) +
                     pool_attr(c->big_pool, cudaMemPoolAttrReservedMemCurrent);
}
// Bytes this context can still allocate: free memory at the snapshot plus
// what its pools had reserved then, minus what they hold in use now.
inline size_t mem_available(spg_ctx* c) {
  size_t used = pool_attr(c->pool, cudaMemPoolAttrUsedMemCurrent) +
                pool_attr(c->big_pool, cudaMemPoolAttrUsedMemCurrent);
  used = used > c->big_cached ? used - c->big_cached : 0;  // cached blocks are ours to reuse
  const size_t have = c->free_snap + c->reserved_snap;
  return have > used ? have - used : 0;
}
inline void dfree(spg_ctx* c, void* p) { dfree_bytes(c, p); }

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
    if (p) {
      try {
        dfree_bytes(c, p);
      } catch (...) {  // destructors must not throw
      }
    }
    p = nullptr;
  }
  T* release() { T* q = p; p = nullptr; return q; }
  static DBuf adopt(spg_ctx* ctx, T* q, size_t count) {
    DBuf b;
    b.c = ctx;
    b.p = q;
    b.n = count;
    return b;
  }
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
