// The extern "C" boundary (include/spgemm_b200.h): contexts, device
// matrices, the local multiply / merge / checksum / slice / prepare entry
// points and the host-array drop-ins.  Every function converts C++
// exceptions into an SPG_ERR_* status + last-error message.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "comm.h"
#include "instantiate.cuh"
#include "layout.cuh"

extern "C" const spg::SrOps* spg_ops_arithmetic();
extern "C" const spg::SrOps* spg_ops_minplus();
extern "C" const spg::SrOps* spg_ops_boolean();
extern "C" const spg::SrOps* spg_ops_minselect();
extern "C" const spg::SrOps* spg_ops_tropical_i32();
extern "C" const spg::SrOps* spg_ops_maxtimes();

namespace spg {
void gen_rmat(int, int, double, uint64_t, int64_t*, int64_t*, int64_t**, int64_t**, void**);
void widen_i32_to_i64(const int32_t* in, int64_t* out, int64_t n);  // hostwiden.cpp
void gen_er(int, int64_t, int, uint64_t, int, int64_t, int64_t, int64_t, int64_t, int64_t*, int64_t**, int64_t**,
            void**);
void gen_stencil27(int, int64_t, int64_t, int64_t, int64_t, int64_t, int64_t*, int64_t*, int64_t**, int64_t**, void**);
void read_matrix_market(int, const char*, int64_t*, int64_t*, int64_t*, int64_t**, int64_t**, void**);

thread_local std::string g_last_error;

// Semiring registry: the built-ins, then user semirings registered at run
// time (ids SPG_SR_COUNT, SPG_SR_COUNT + 1, ...; append-only).
std::mutex g_sr_mu;
std::vector<const SrOps*> g_sr_user;

const SrOps* ops_for(int sr) {
  switch (sr) {
    case SPG_SR_ARITHMETIC: return spg_ops_arithmetic();
    case SPG_SR_MINPLUS: return spg_ops_minplus();
    case SPG_SR_BOOLEAN: return spg_ops_boolean();
    case SPG_SR_MINSELECT: return spg_ops_minselect();
    case SPG_SR_TROPICAL_I32: return spg_ops_tropical_i32();
    case SPG_SR_MAXTIMES: return spg_ops_maxtimes();
  }
  if (sr >= SPG_SR_COUNT) {
    std::lock_guard<std::mutex> g(g_sr_mu);
    if ((size_t)(sr - SPG_SR_COUNT) < g_sr_user.size()) return g_sr_user[(size_t)(sr - SPG_SR_COUNT)];
  }
  fail(SPG_ERR_ARG, "unknown semiring id " + std::to_string(sr));
}

int semiring_count() {
  std::lock_guard<std::mutex> g(g_sr_mu);
  return SPG_SR_COUNT + (int)g_sr_user.size();
}

template <class F>
int guarded(spg_ctx* c, F&& f) {
  try {
    f();
    return SPG_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    if (c) c->last_error = e.what();
    return e.status;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    if (c) c->last_error = g_last_error;
    return SPG_ERR_OOM;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    if (c) c->last_error = e.what();
    return SPG_ERR_INTERNAL;
  }
}

// Runs one rank's distributed program.  Validation errors are symmetric
// across ranks and leave the fabric usable; anything raised after the first
// collective tears the peers down (AbortedError on their side).
int guarded_summa(spg_ctx* c, spg_comm* comm, const std::function<void()>& f) {
  const int rc = guarded(c, f);
  if (rc != SPG_OK && comm && rc != SPG_ERR_ABORTED && rc != SPG_ERR_DEADLOCK && rc != SPG_ERR_SHAPE &&
      rc != SPG_ERR_UNSUPPORTED_SEMIRING && rc != SPG_ERR_ARG && rc != SPG_ERR_GRID)
    comm_abort(comm, c ? c->last_error : g_last_error);
  return rc;
}

void need(bool ok, const char* what) {
  if (!ok) fail(SPG_ERR_ARG, what);
}

void use_device(spg_ctx* c) { SPG_CUDA(cudaSetDevice(c->device)); }

void upload_indices(spg_ctx* c, const int64_t* h, int32_t* d, int64_t n, int64_t bound);  // below

// Host CSR/CSC -> device (int64 indices narrowed to int32 on the way).
void upload(spg_ctx* c, int vs, const spg_hcsr* h, int is_csc, spg_dcsr* d) {
  const int64_t nseg = is_csc ? h->ncols : h->nrows;
  const int64_t bound = is_csc ? h->nrows : h->ncols;
  need(h->nrows >= 0 && h->ncols >= 0 && h->nnz >= 0, "negative dims");
  if (bound > INT32_MAX) fail(SPG_ERR_INVALID_RANGE, "block dimension exceeds int32 indices");
  if (h->ptr == nullptr) fail(SPG_ERR_ARG, "null offsets");
  if (h->ptr[0] != 0 || h->ptr[nseg] != h->nnz)
    fail(SPG_ERR_MALFORMED, "offset array is not a monotone [0..nnz] map");
  d->nrows = h->nrows;
  d->ncols = h->ncols;
  d->nnz = h->nnz;
  d->ptr = dalloc<int64_t>(c, nseg + 1);
  d->idx = dalloc<int32_t>(c, h->nnz);
  d->vals = dalloc<char>(c, (size_t)vs * h->nnz);
  SPG_CUDA(cudaMemcpyAsync(d->ptr, h->ptr, sizeof(int64_t) * (nseg + 1), cudaMemcpyHostToDevice, c->stream));
  if (h->nnz > 0) {
    // values first: their copy runs while host threads narrow the first index chunks
    SPG_CUDA(cudaMemcpyAsync(d->vals, h->vals, (size_t)vs * h->nnz, cudaMemcpyHostToDevice, c->stream));
    upload_indices(c, h->idx, d->idx, h->nnz, bound);
  }
}

// Caching allocator of pinned host memory for results (D2H at full PCIe
// speed; page-locking tens of GB per call would cost seconds).  Blocks are
// recycled by size class; anything not from the cache is plain malloc.
struct PinnedCache {
  std::mutex mu;
  std::multimap<size_t, void*> free_blocks;
  std::map<void*, size_t> live;
  size_t cached_bytes = 0;

  static size_t round_up(size_t n) {
    size_t c = 1 << 20;
    while (c < n) c <<= 1;
    return c;
  }
  void* get(size_t n) {
    const size_t cls = round_up(std::max<size_t>(n, 1));
    {
      std::lock_guard<std::mutex> g(mu);
      auto it = free_blocks.lower_bound(cls);
      if (it != free_blocks.end() && it->first == cls) {
        void* p = it->second;
        free_blocks.erase(it);
        cached_bytes -= cls;
        live[p] = cls;
        return p;
      }
    }
    void* p = nullptr;
    HostTrace ht("cudaHostAlloc", cls);
    if (cudaHostAlloc(&p, cls, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      if (HostTrace::limit_ms() >= 0) std::fprintf(stderr, "[spg-host] cudaHostAlloc(%zu) refused: pageable\n", cls);
      p = std::malloc(n);  // fall back to pageable memory
      if (!p) fail(SPG_ERR_OOM, "host allocation failed");
      return p;
    }
    std::lock_guard<std::mutex> g(mu);
    live[p] = cls;
    return p;
  }
  // returns true when p was a cached pinned block
  bool put(void* p) {
    if (!p) return true;
    std::lock_guard<std::mutex> g(mu);
    auto it = live.find(p);
    if (it == live.end()) return false;
    const size_t cls = it->second;
    live.erase(it);
    // keep at most 64 GB cached; release the rest
    if (cached_bytes + cls > (size_t(64) << 30)) {
      cudaFreeHost(p);
      return true;
    }
    free_blocks.emplace(cls, p);
    cached_bytes += cls;
    return true;
  }
};

PinnedCache& pinned() {
  static PinnedCache* pc = new PinnedCache();  // intentionally leaked: outlives late frees
  return *pc;
}

void host_release(void* p) {
  if (!pinned().put(p)) std::free(p);
}



// Persistent host worker pool: parallel_for(n, fn) runs fn(lo, hi) over n
// items split across the workers and the caller, and returns when all are done.
// Calls from several host threads (one context per GPU) are serialised by
// call_mu_: a job owns the pool until every part has finished.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool* p = new HostPool();  // intentionally leaked (process lifetime)
    return *p;
  }
  void parallel_for(int64_t n, const std::function<void(int64_t, int64_t)>& fn) {
    std::lock_guard<std::mutex> call(call_mu_);
    const int parts = (int)workers_.size() + 1;
    std::unique_lock<std::mutex> lk(mu_);
    job_ = &fn;
    n_ = n;
    parts_ = parts;
    pending_ = parts - 1;
    ++gen_;
    cv_.notify_all();
    lk.unlock();
    fn(0, n / parts);  // the caller takes part 0
    lk.lock();
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
  }

 private:
  HostPool() {
    const int t = (int)std::max(1u, std::min(32u, std::thread::hardware_concurrency())) - 1;
    for (int k = 0; k < t; ++k) workers_.emplace_back([this, k] { run(k + 1); });
    for (auto& w : workers_) w.detach();
  }
  void run(int part) {
    uint64_t seen = 0;
    for (;;) {
      std::unique_lock<std::mutex> lk(mu_);
      cv_.wait(lk, [&] { return gen_ != seen; });
      seen = gen_;
      const auto* fn = job_;
      const int64_t n = n_;
      const int parts = parts_;
      lk.unlock();
      (*fn)(n * part / parts, n * (part + 1) / parts);
      lk.lock();
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::vector<std::thread> workers_;
  std::mutex call_mu_;  // one parallel_for at a time
  std::mutex mu_;
  std::condition_variable cv_, done_;
  const std::function<void(int64_t, int64_t)>* job_ = nullptr;
  int64_t n_ = 0;
  int parts_ = 1, pending_ = 0;
  uint64_t gen_ = 0;
};

// share of index chunks widened on the GPU (the rest cross PCIe as int32 and
// are widened by host threads with streaming stores, hostwiden.cpp):
// config-2 e2e 0.301 s at 0, 0.270-0.276 s at 0.1, 0.272-0.281 s at 0.2,
// 0.305-0.355 s at 1 (all int64 on the bus: PCIe bound)
constexpr double kGpuWiden = 0.1;

bool narrow_i64_to_i32(const int64_t* in, int32_t* out, int64_t n, int64_t bound);  // hostwiden.cpp

// processes of this job on this host (set by spg_comm_create; 1 without a communicator)
std::atomic<int> g_host_procs{1};
void note_host_procs(int n) { g_host_procs.store(n > 1 ? n : 1); }

// int64 host indices -> int32 device indices.  Large arrays cross PCIe as
// int32: host threads narrow (and range-check) 2^25-entry chunks into two
// pinned staging buffers while the previous chunk is in flight — half the
// bytes on the bus.  Small arrays (and SPG_H2D_HOST_NARROW=0) go as int64 and
// are narrowed by a device kernel.  MalformedInputError on an index outside
// [0, bound) either way.
void upload_indices(spg_ctx* c, const int64_t* h, int32_t* d, int64_t n, int64_t bound) {
  if (n <= 0) return;
  static const int host_narrow = [] {
    const char* e = std::getenv("SPG_H2D_HOST_NARROW");
    return e ? std::atoi(e) : 1;
  }();
  // (several processes of a job on this host: their threads would share its
  // memory bandwidth, so the indices go as int64 and narrow on each GPU)
  if (!host_narrow || n < (int64_t(1) << 22) || g_host_procs.load() > 1) {
    DBuf<int64_t> wide(c, n);
    SPG_CUDA(cudaMemcpyAsync(wide.p, h, sizeof(int64_t) * n, cudaMemcpyHostToDevice, c->stream));
    narrow_indices(c, wide.p, d, n, bound);
    return;
  }
  const int64_t chunk = std::min<int64_t>(int64_t(1) << 25, n);
  int32_t* stage[2] = {static_cast<int32_t*>(pinned().get(sizeof(int32_t) * chunk)),
                       static_cast<int32_t*>(pinned().get(sizeof(int32_t) * chunk))};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  std::atomic<bool> bad{false};
  auto cleanup = [&] {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    host_release(stage[0]);
    host_release(stage[1]);
  };
  try {
    for (auto& e : ev) SPG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const int64_t nch = (n + chunk - 1) / chunk;
    for (int64_t k = 0; k < nch; ++k) {
      const int64_t o = k * chunk, m = std::min<int64_t>(chunk, n - o);
      const int slot = (int)(k & 1);
      if (k >= 2) SPG_CUDA(cudaEventSynchronize(ev[slot]));  // the copy out of this stage is done
      int32_t* st = stage[slot];
      HostPool::get().parallel_for(m, [&](int64_t lo, int64_t hi) {
        if (!narrow_i64_to_i32(h + o + lo, st + lo, hi - lo, bound)) bad = true;
      });
      SPG_CUDA(cudaMemcpyAsync(d + o, st, sizeof(int32_t) * m, cudaMemcpyHostToDevice, c->stream));
      SPG_CUDA(cudaEventRecord(ev[slot], c->stream));
    }
    SPG_CUDA(cudaStreamSynchronize(c->stream));
  } catch (...) {
    cudaStreamSynchronize(c->stream);
    cleanup();
    throw;
  }
  cleanup();
  if (bad) fail(SPG_ERR_MALFORMED, "index outside [0, " + std::to_string(bound) + ")");
}

void download(spg_ctx* c, int vs, const spg_dcsr* d, int is_csc, spg_hcsr* h) {
  const int64_t nseg = is_csc ? d->ncols : d->nrows;
  h->nrows = d->nrows;
  h->ncols = d->ncols;
  h->nnz = d->nnz;
  h->ptr = static_cast<int64_t*>(pinned().get(sizeof(int64_t) * (nseg + 1)));
  h->idx = static_cast<int64_t*>(pinned().get(sizeof(int64_t) * std::max<int64_t>(d->nnz, 1)));
  h->vals = pinned().get((size_t)vs * std::max<int64_t>(d->nnz, 1));
  SPG_CUDA(cudaMemcpyAsync(h->ptr, d->ptr, sizeof(int64_t) * (nseg + 1), cudaMemcpyDeviceToHost, c->stream));
  if (d->nnz > 0) {
    // int32 indices cross PCIe in chunks through two pinned staging buffers
    // and are widened to the reference's int64 by host threads while the
    // next chunk (and finally the values) is in flight: 4 + V bytes per
    // entry on the bus instead of 8 + V.  A fraction of the chunks
    // (SPG_D2H_GPU_WIDEN, default kGpuWiden) is widened on the GPU and crosses
    // as int64 instead, balancing PCIe bytes against host memory bandwidth.
    const int64_t chunk = std::min<int64_t>(int64_t(1) << 25, d->nnz);
    int32_t* stage[2] = {static_cast<int32_t*>(pinned().get(sizeof(int32_t) * chunk)),
                         static_cast<int32_t*>(pinned().get(sizeof(int32_t) * chunk))};
    cudaEvent_t ev[2];
    for (auto& e : ev) SPG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    static const double env_frac = [] {
      const char* e = std::getenv("SPG_D2H_GPU_WIDEN");
      const double f = e ? std::atof(e) : -1.0;
      return f < 0 && e ? 0.0 : f > 1 ? 1.0 : f;
    }();
    // several processes of a job on this host (one per GPU) would share its
    // memory bandwidth for the widening: then every chunk widens on its GPU
    // (1x2 config-2 e2e 0.171 s with host widening, 0.148 s on the GPUs)
    const double gpu_frac = env_frac >= 0 ? env_frac : (g_host_procs.load() > 1 ? 1.0 : kGpuWiden);
    DBuf<int64_t> dwide[2];
    double frac = gpu_frac;
    if (frac > 0) {  // no room for the two device staging buffers: widen everything on the host
      for (auto& b : dwide) {
        int64_t* p = try_dalloc<int64_t>(c, (size_t)chunk);
        if (!p) {
          frac = 0;
          break;
        }
        b = DBuf<int64_t>::adopt(c, p, (size_t)chunk);
      }
    }
    auto widen = [&](int k, int slot) {
      const int64_t o = (int64_t)k * chunk, n = std::min<int64_t>(chunk, d->nnz - o);
      {
        HostTrace ht("download: wait chunk", (size_t)k);
        SPG_CUDA(cudaEventSynchronize(ev[slot]));
      }
      const int32_t* in = stage[slot];
      int64_t* out = h->idx + o;
      HostTrace ht("download: widen chunk", (size_t)k);
      HostPool::get().parallel_for(n, [&](int64_t lo, int64_t hi) { widen_i32_to_i64(in + lo, out + lo, hi - lo); });
    };
    const int nch = (int)((d->nnz + chunk - 1) / chunk);
    // values on a side stream, concurrently with the index pipeline
    cudaStream_t side = nullptr;
    cudaEvent_t ready = nullptr;
    SPG_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    SPG_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    SPG_CUDA(cudaEventRecord(ready, c->stream));
    SPG_CUDA(cudaStreamWaitEvent(side, ready, 0));
    SPG_CUDA(cudaMemcpyAsync(h->vals, d->vals, (size_t)vs * d->nnz, cudaMemcpyDeviceToHost, side));
    try {
      int hosted = 0, gpu = 0, pending = -1, pending_slot = 0;
      for (int k = 0; k < nch; ++k) {
        const int64_t o = (int64_t)k * chunk, n = std::min<int64_t>(chunk, d->nnz - o);
        // Bresenham spread: chunk k goes wide on the GPU when the running share falls behind gpu_frac
        if (frac > 0 && (double)(gpu + 1) <= frac * (double)(k + 1) + 1e-9) {
          widen_indices(c, d->idx + o, dwide[gpu & 1].p, n);
          SPG_CUDA(cudaMemcpyAsync(h->idx + o, dwide[gpu & 1].p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost,
                                   c->stream));
          ++gpu;
          continue;
        }
        const int slot = hosted & 1;
        SPG_CUDA(cudaMemcpyAsync(stage[slot], d->idx + o, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
        SPG_CUDA(cudaEventRecord(ev[slot], c->stream));
        if (pending >= 0) widen(pending, pending_slot);  // the chunk before this one (its slot is the other)
        pending = k;
        pending_slot = slot;
        ++hosted;
      }
      if (pending >= 0) widen(pending, pending_slot);
      SPG_CUDA(cudaStreamSynchronize(side));
    } catch (...) {
      cudaStreamSynchronize(side);
      cudaStreamDestroy(side);
      cudaEventDestroy(ready);
      for (auto& e : ev) cudaEventDestroy(e);
      host_release(stage[0]);
      host_release(stage[1]);
      throw;
    }
    cudaStreamDestroy(side);
    cudaEventDestroy(ready);
    for (auto& e : ev) cudaEventDestroy(e);
    host_release(stage[0]);
    host_release(stage[1]);
  }
  HostTrace ht("download sync", (size_t)d->nnz);
  SPG_CUDA(cudaStreamSynchronize(c->stream));
}

void free_dcsr(spg_ctx* c, spg_dcsr* m) {
  dfree(c, m->ptr);
  dfree(c, m->idx);
  dfree(c, m->vals);
  m->ptr = nullptr;
  m->idx = nullptr;
  m->vals = nullptr;
}

}  // namespace spg

using namespace spg;

extern "C" {

const char* spg_version(void) { return "spgemm_b200 0.1 (sm_100a)"; }

const char* spg_last_error(const spg_ctx* ctx) {
  return ctx ? ctx->last_error.c_str() : g_last_error.c_str();
}

int spg_value_size(int sr) {
  try {
    return ops_for(sr)->value_size;
  } catch (...) {
    return -1;
  }
}

int spg_semiring_by_name(const char* name) {
  if (!name) return -1;
  const int n = semiring_count();
  for (int s = 0; s < n; ++s)
    if (std::strcmp(name, ops_for(s)->name) == 0) return s;
  g_last_error = std::string("unknown semiring '") + name +
                 "' (expected arithmetic, minplus, boolean, minselect, tropical_i32, or maxtimes)";
  return -1;
}

int spg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int spg_register_semiring(const spg_semiring_ops* ops_in, int* id) {
  return guarded(nullptr, [&] {
    const SrOps* ops = reinterpret_cast<const SrOps*>(ops_in);
    need(ops && id, "null argument");
    if (ops->abi != kSrOpsAbi)
      fail(SPG_ERR_ARG, "semiring ops table ABI " + std::to_string(ops->abi) + " != " + std::to_string(kSrOpsAbi) +
                            " (rebuild the semiring library against this release's headers)");
    need(ops->name && ops->name[0] && ops->local_multiply && ops->merge && ops->checksum_part &&
             ops->fold_runs,
         "incomplete semiring ops table");
    if (ops->value_size != 1 && ops->value_size != 2 && ops->value_size != 4 && ops->value_size != 8 &&
        ops->value_size != 16)
      fail(SPG_ERR_ARG, "semiring value size must be 1, 2, 4, 8 or 16 bytes");
    std::lock_guard<std::mutex> g(g_sr_mu);
    for (int s = 0; s < SPG_SR_COUNT; ++s)
      if (std::strcmp(ops_for(s)->name, ops->name) == 0)
        fail(SPG_ERR_ARG, std::string("semiring name '") + ops->name + "' is a built-in");
    for (size_t k = 0; k < g_sr_user.size(); ++k) {
      if (g_sr_user[k] == ops) {  // registering the same table again returns its id
        *id = SPG_SR_COUNT + (int)k;
        return;
      }
      if (std::strcmp(g_sr_user[k]->name, ops->name) == 0)
        fail(SPG_ERR_ARG, std::string("a different semiring named '") + ops->name + "' is already registered");
    }
    g_sr_user.push_back(ops);
    *id = SPG_SR_COUNT + (int)g_sr_user.size() - 1;
  });
}

const char* spg_semiring_name(int sr) {
  try {
    return ops_for(sr)->name;
  } catch (...) {
    return nullptr;
  }
}

int spg_semiring_is_commutative(int sr) {
  try {
    return ops_for(sr)->commutative ? 1 : 0;
  } catch (...) {
    return -1;
  }
}

int spg_ctx_create(int device, spg_ctx** out) {
  return guarded(nullptr, [&] {
    need(out != nullptr, "null out");
    auto* c = new spg_ctx();
    try {
      c->device = device;
      SPG_CUDA(cudaSetDevice(device));
      SPG_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
      SPG_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
      SPG_CUDA(cudaDeviceGetDefaultMemPool(&c->pool, device));
      uint64_t thr = UINT64_MAX;  // keep freed blocks cached in the pool
      SPG_CUDA(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &thr));
      cudaMemPoolProps props{};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = device;
      SPG_CUDA(cudaMemPoolCreate(&c->big_pool, &props));
      SPG_CUDA(cudaMemPoolSetAttribute(c->big_pool, cudaMemPoolAttrReleaseThreshold, &thr));
      mem_snapshot(c);
    } catch (...) {
      if (c->big_pool) cudaMemPoolDestroy(c->big_pool);
      delete c;
      throw;
    }
    *out = c;
  });
}

void spg_ctx_destroy(spg_ctx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->cub_tmp) cudaFreeAsync(c->cub_tmp, c->stream);
  for (auto& kv : c->big_free) cudaFreeAsync(kv.second, c->stream);
  c->big_free.clear();
  cudaStreamSynchronize(c->stream);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (int k = 0; k < 4; ++k) {
    if (c->aux[k]) cudaStreamDestroy(c->aux[k]);
    if (c->aux_ev[k]) cudaEventDestroy(c->aux_ev[k]);
  }
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  if (c->big_pool) {
    cudaDeviceSynchronize();  // buffers the caller freed stream-ordered must be back in the pool
    cudaMemPoolDestroy(c->big_pool);
  }
  delete c;
}

void* spg_ctx_stream(spg_ctx* c) { return c ? (void*)c->stream : nullptr; }

int spg_ctx_set_stream(spg_ctx* c, void* stream) {
  return guarded(c, [&] {
    need(c != nullptr, "null ctx");
    SPG_CUDA(cudaStreamSynchronize(c->stream));
    if (c->own_stream) SPG_CUDA(cudaStreamDestroy(c->stream));
    c->stream = static_cast<cudaStream_t>(stream);
    c->own_stream = false;
  });
}

int spg_ctx_sync(spg_ctx* c) {
  return guarded(c, [&] { SPG_CUDA(cudaStreamSynchronize(c->stream)); });
}

uint64_t spg_ctx_kernel_launches(const spg_ctx* c) { return c ? c->launches : 0; }

int spg_ctx_set_scratch_budget(spg_ctx* c, uint64_t bytes) {
  return guarded(c, [&] { c->scratch_budget = bytes; });
}

int spg_ctx_set_pipeline(spg_ctx* c, int mode) {
  return guarded(c, [&] {
    need(c && (mode == SPG_PIPE_AUTO || mode == SPG_PIPE_BINS || mode == SPG_PIPE_SORTED), "pipeline: unknown mode");
    c->pipeline = mode;
  });
}

int spg_dcsr_alloc(spg_ctx* c, int sr, int64_t nrows, int64_t ncols, int64_t nseg, int64_t nnz, spg_dcsr* out) {
  return guarded(c, [&] {
    need(c && out, "null argument");
    use_device(c);
    const int vs = ops_for(sr)->value_size;
    out->nrows = nrows;
    out->ncols = ncols;
    out->nnz = nnz;
    out->ptr = dalloc<int64_t>(c, nseg + 1);
    out->idx = dalloc<int32_t>(c, nnz);
    out->vals = dalloc<char>(c, (size_t)vs * nnz);
  });
}

int spg_dcsr_free(spg_ctx* c, spg_dcsr* m) {
  return guarded(c, [&] {
    need(c && m, "null argument");
    use_device(c);
    free_dcsr(c, m);
  });
}

int spg_copy_to_host(spg_ctx* c, void* dst, const void* src, uint64_t bytes) {
  return guarded(c, [&] {
    need(c && (bytes == 0 || (dst && src)), "null argument");
    use_device(c);
    if (bytes) SPG_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, c->stream));
    SPG_CUDA(cudaStreamSynchronize(c->stream));
  });
}

int spg_upload(spg_ctx* c, int sr, const spg_hcsr* h, int is_csc, spg_dcsr* out) {
  return guarded(c, [&] {
    need(c && h && out, "null argument");
    use_device(c);
    upload(c, ops_for(sr)->value_size, h, is_csc, out);
  });
}

int spg_download(spg_ctx* c, int sr, const spg_dcsr* d, int is_csc, spg_hcsr* out) {
  return guarded(c, [&] {
    need(c && d && out, "null argument");
    use_device(c);
    download(c, ops_for(sr)->value_size, d, is_csc, out);
  });
}

void spg_hcsr_free(spg_hcsr* h) {
  if (!h) return;
  host_release(h->ptr);
  host_release(h->idx);
  host_release(h->vals);
  h->ptr = nullptr;
  h->idx = nullptr;
  h->vals = nullptr;
}

int spg_local_multiply(spg_ctx* c, int sr, const spg_dcsr* a, const spg_dcsr* b, spg_dcsr* out,
                       spg_mult_stats* st) {
  return guarded(c, [&] {
    need(c && a && b && out, "null argument");
    use_device(c);
    // local_spgemm.hpp:14-21
    if (a->ncols != b->nrows)
      fail(SPG_ERR_SHAPE, "cannot multiply " + std::to_string(a->nrows) + "x" + std::to_string(a->ncols) +
                              " by " + std::to_string(b->nrows) + "x" + std::to_string(b->ncols));
    if (b->ncols > INT32_MAX) fail(SPG_ERR_INVALID_RANGE, "output width exceeds int32 indices");
    ops_for(sr)->local_multiply(c, a, b, out, st);
  });
}

int spg_local_multiply_rows(spg_ctx* c, int sr, const spg_dcsr* a, const spg_dcsr* b, int64_t row_begin,
                            int64_t row_end, spg_dcsr* out, spg_mult_stats* st) {
  return guarded(c, [&] {
    need(c && a && b && out, "null argument");
    use_device(c);
    if (a->ncols != b->nrows)
      fail(SPG_ERR_SHAPE, "cannot multiply " + std::to_string(a->nrows) + "x" + std::to_string(a->ncols) +
                              " by " + std::to_string(b->nrows) + "x" + std::to_string(b->ncols));
    if (row_begin < 0 || row_end < row_begin || row_end > a->nrows)
      fail(SPG_ERR_INVALID_RANGE, "row range [" + std::to_string(row_begin) + ", " + std::to_string(row_end) +
                                      ") outside 0.." + std::to_string(a->nrows));
    if (b->ncols > INT32_MAX) fail(SPG_ERR_INVALID_RANGE, "output width exceeds int32 indices");
    spg_dcsr v = *a;  // row window: the row pointers index the whole operand's entries
    v.nrows = row_end - row_begin;
    v.ptr = a->ptr + row_begin;
    ops_for(sr)->local_multiply(c, &v, b, out, st);
  });
}

int spg_merge_partials(spg_ctx* c, int sr, int nparts, const spg_dcsr* parts, const int* stages,
                       const int* rounds, int64_t block_rows, int64_t block_cols, spg_dcsr* out,
                       spg_mult_stats* st) {
  return guarded(c, [&] {
    need(c && out && (nparts == 0 || parts), "null argument");
    use_device(c);
    std::vector<int> order(nparts);
    for (int i = 0; i < nparts; ++i) order[i] = i;
    if (stages && rounds)  // stable (stage, round) order, summa.hpp:125-129
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
        return stages[x] != stages[y] ? stages[x] < stages[y] : rounds[x] < rounds[y];
      });
    std::vector<spg_dcsr> ps;
    for (int i : order) {
      const spg_dcsr& p = parts[i];
      if (p.nrows != block_cols || p.ncols != block_rows)  // summa.hpp:133-138
        fail(SPG_ERR_INTERNAL, "partial extents " + std::to_string(p.nrows) + "x" + std::to_string(p.ncols) +
                                   " do not match the " + std::to_string(block_rows) + "x" +
                                   std::to_string(block_cols) + " output block");
      ps.push_back(p);
    }
    // CSR of C^T (block_cols x block_rows) == CSC of C
    ops_for(sr)->merge(c, nparts, ps.data(), block_cols, block_rows, out, st);
    out->nrows = block_rows;
    out->ncols = block_cols;
  });
}

int spg_checksum(spg_ctx* c, int sr, const spg_dcsr* m, int is_csc, uint64_t* out) {
  return guarded(c, [&] {
    need(c && m && out, "null argument");
    use_device(c);
    *out = splitmix64((uint64_t)m->nrows * 31 + (uint64_t)m->ncols) + ops_for(sr)->checksum_part(c, m, is_csc, 0, 0);
  });
}

int spg_checksum_part(spg_ctx* c, int sr, const spg_dcsr* m, int is_csc, int64_t row_off, int64_t col_off,
                      uint64_t* out) {
  return guarded(c, [&] {
    need(c && m && out, "null argument");
    use_device(c);
    *out = ops_for(sr)->checksum_part(c, m, is_csc, row_off, col_off);
  });
}

uint64_t spg_checksum_seed(int64_t nrows, int64_t ncols) {
  return splitmix64((uint64_t)nrows * 31 + (uint64_t)ncols);
}

int spg_csr_slice(spg_ctx* c, int sr, const spg_dcsr* m, int by_rows, int64_t begin, int64_t end,
                  spg_dcsr* out) {
  return guarded(c, [&] {
    need(c && m && out, "null argument");
    use_device(c);
    const int vs = ops_for(sr)->value_size;
    const int64_t lim = by_rows ? m->nrows : m->ncols;
    if (begin < 0 || end < begin || end > lim) fail(SPG_ERR_INVALID_RANGE, "slice range outside the matrix");
    if (by_rows) {
      int64_t lo = 0, hi = 0;
      SPG_CUDA(cudaMemcpyAsync(&lo, m->ptr + begin, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
      SPG_CUDA(cudaMemcpyAsync(&hi, m->ptr + end, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
      SPG_CUDA(cudaStreamSynchronize(c->stream));
      out->nrows = end - begin;
      out->ncols = m->ncols;
      out->nnz = hi - lo;
      out->ptr = dalloc<int64_t>(c, end - begin + 1);
      out->idx = dalloc<int32_t>(c, hi - lo);
      out->vals = dalloc<char>(c, (size_t)vs * (hi - lo));
      slice_rows_into(c, *m, begin, end, vs, *out);
    } else {
      out->nrows = m->nrows;
      out->ncols = end - begin;
      out->ptr = dalloc<int64_t>(c, m->nrows + 1);
      DBuf<int64_t> cnt(c, m->nrows + 1);
      slice_cols_count(c, *m, begin, end, cnt.p);
      exclusive_scan_i64(c, cnt.p, out->ptr, m->nrows + 1);
      out->nnz = d2h_scalar(c, out->ptr + m->nrows);
      out->idx = dalloc<int32_t>(c, out->nnz);
      out->vals = dalloc<char>(c, (size_t)vs * out->nnz);
      slice_cols_fill(c, *m, begin, end, vs, *out);
    }
  });
}

}  // extern "C"

namespace spg {

// prepare_block (summa.hpp:30-53): device CSR of the block's transpose.
void prepare_block(spg_ctx* c, int sr, const spg_hcsr* csc, const spg_hdcsc* dcsc, spg_dcsr* out) {
  const SrOps* ops = ops_for(sr);
  if (!ops->commutative)
    fail(SPG_ERR_UNSUPPORTED_SEMIRING,
         std::string("semiring '") + ops->name +
             "' has a non-commutative multiplication; the distributed transpose-reinterpretation path "
             "supports commutative semirings only");
  const int vs = ops->value_size;
  if (dcsc) {
    // dcsc_decompress checks (formats.hpp:222-242), done on the host arrays
    // cp always has njc + 1 entries (njc == 0 included); jc has njc
    if (dcsc->njc < 0 || !dcsc->cp || (dcsc->njc > 0 && !dcsc->jc))
      fail(SPG_ERR_MALFORMED, "dcsc_decompress: bad cp offset array");
    if (dcsc->cp[0] != 0 || dcsc->cp[dcsc->njc] != dcsc->nnz)
      fail(SPG_ERR_MALFORMED, "dcsc_decompress: bad cp offset array");
    int64_t prev = -1;
    for (int64_t i = 0; i < dcsc->njc; ++i) {
      if (dcsc->cp[i + 1] < dcsc->cp[i]) fail(SPG_ERR_MALFORMED, "dcsc_decompress: bad cp offset array");
      const int64_t col = dcsc->jc[i];
      if (col <= prev || col >= dcsc->ncols)
        fail(SPG_ERR_MALFORMED, "dcsc_decompress: jc column id " + std::to_string(col) +
                                    " out of range or not strictly increasing");
      prev = col;
    }
    if (dcsc->nrows > INT32_MAX) fail(SPG_ERR_INVALID_RANGE, "block dimension exceeds int32 indices");
    // transposed view: rows = block cols, cols = block rows
    out->nrows = dcsc->ncols;
    out->ncols = dcsc->nrows;
    out->nnz = dcsc->nnz;
    out->ptr = dalloc<int64_t>(c, dcsc->ncols + 1);
    out->idx = dalloc<int32_t>(c, dcsc->nnz);
    out->vals = dalloc<char>(c, (size_t)vs * dcsc->nnz);
    DBuf<int64_t> jc(c, dcsc->njc), cp(c, dcsc->njc + 1);
    if (dcsc->njc > 0)
      SPG_CUDA(cudaMemcpyAsync(jc.p, dcsc->jc, sizeof(int64_t) * dcsc->njc, cudaMemcpyHostToDevice, c->stream));
    SPG_CUDA(cudaMemcpyAsync(cp.p, dcsc->cp, sizeof(int64_t) * (dcsc->njc + 1), cudaMemcpyHostToDevice, c->stream));
    dcsc_colptr(c, dcsc->ncols, dcsc->njc, jc.p, cp.p, out->ptr);
    if (dcsc->nnz > 0) {
      SPG_CUDA(cudaMemcpyAsync(out->vals, dcsc->vals, (size_t)vs * dcsc->nnz, cudaMemcpyHostToDevice, c->stream));
      upload_indices(c, dcsc->rowids, out->idx, dcsc->nnz, dcsc->nrows);
    }
  } else {
    spg_dcsr d{};
    upload(c, vs, csc, /*is_csc=*/1, &d);
    // reinterpret_transpose (formats.hpp:255-264): the CSC arrays read as CSR
    out->nrows = csc->ncols;
    out->ncols = csc->nrows;
    out->nnz = csc->nnz;
    out->ptr = d.ptr;
    out->idx = d.idx;
    out->vals = d.vals;
  }
}

}  // namespace spg

extern "C" {

int spg_prepare_block(spg_ctx* c, int sr, const spg_hcsr* csc, const spg_hdcsc* dcsc, spg_dcsr* prepared) {
  return guarded(c, [&] {
    need(c && prepared && (csc || dcsc), "null argument");
    use_device(c);
    prepare_block(c, sr, csc, dcsc, prepared);
  });
}

int spg_esc_multiply(spg_ctx* c, int sr, const spg_hcsr* a, const spg_hcsr* b, spg_hcsr* out,
                     spg_mult_stats* st) {
  return guarded(c, [&] {
    need(c && a && b && out, "null argument");
    use_device(c);
    if (a->ncols != b->nrows)
      fail(SPG_ERR_SHAPE, "cannot multiply " + std::to_string(a->nrows) + "x" + std::to_string(a->ncols) +
                              " by " + std::to_string(b->nrows) + "x" + std::to_string(b->ncols));
    const SrOps* ops = ops_for(sr);
    spg_dcsr da{}, db{}, dc{};
    {
      HostTrace ht("esc upload");
      upload(c, ops->value_size, a, 0, &da);
      upload(c, ops->value_size, b, 0, &db);
      SPG_CUDA(cudaStreamSynchronize(c->stream));
    }
    try {
      {
        HostTrace ht("esc local multiply");
        ops->local_multiply(c, &da, &db, &dc, st);
        SPG_CUDA(cudaStreamSynchronize(c->stream));
      }
      HostTrace ht("esc download");
      download(c, ops->value_size, &dc, 0, out);
    } catch (...) {
      free_dcsr(c, &da);
      free_dcsr(c, &db);
      free_dcsr(c, &dc);
      throw;
    }
    free_dcsr(c, &da);
    free_dcsr(c, &db);
    free_dcsr(c, &dc);
  });
}

int spg_generate_rmat(int sr, int scale, double ef, uint64_t seed, int64_t* nrows, int64_t* nnz, int64_t** rows,
                      int64_t** cols, void** vals) {
  return guarded(nullptr, [&] {
    need(nrows && nnz && rows && cols && vals, "null argument");
    gen_rmat(sr, scale, ef, seed, nrows, nnz, rows, cols, vals);
  });
}

int spg_generate_er(int sr, int64_t n, int d, uint64_t seed, int mode, int64_t* nnz, int64_t** rows,
                    int64_t** cols, void** vals) {
  return guarded(nullptr, [&] {
    need(nnz && rows && cols && vals, "null argument");
    gen_er(sr, n, d, seed, mode, 0, n, 0, n, nnz, rows, cols, vals);
  });
}

int spg_generate_er_block(int sr, int64_t n, int d, uint64_t seed, int mode, int64_t r0, int64_t r1, int64_t c0,
                          int64_t c1, int64_t* nnz, int64_t** rows, int64_t** cols, void** vals) {
  return guarded(nullptr, [&] {
    need(nnz && rows && cols && vals, "null argument");
    gen_er(sr, n, d, seed, mode, r0, r1, c0, c1, nnz, rows, cols, vals);
  });
}

int spg_generate_stencil27(int sr, int64_t N, int64_t* nrows, int64_t* nnz, int64_t** rows, int64_t** cols,
                           void** vals) {
  return guarded(nullptr, [&] {
    need(nrows && nnz && rows && cols && vals, "null argument");
    gen_stencil27(sr, N, 0, N * N * N, 0, N * N * N, nrows, nnz, rows, cols, vals);
  });
}

int spg_generate_stencil27_block(int sr, int64_t N, int64_t r0, int64_t r1, int64_t c0, int64_t c1, int64_t* nrows,
                                 int64_t* nnz, int64_t** rows, int64_t** cols, void** vals) {
  return guarded(nullptr, [&] {
    need(nrows && nnz && rows && cols && vals, "null argument");
    gen_stencil27(sr, N, r0, r1, c0, c1, nrows, nnz, rows, cols, vals);
  });
}

int spg_read_matrix_market(int sr, const char* path, int64_t* nrows, int64_t* ncols, int64_t* nnz, int64_t** rows,
                           int64_t** cols, void** vals) {
  return guarded(nullptr, [&] {
    need(path && nrows && ncols && nnz && rows && cols && vals, "null argument");
    read_matrix_market(sr, path, nrows, ncols, nnz, rows, cols, vals);
  });
}

int spg_coo_to_csr(int sr, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows, const int64_t* cols,
                   const void* vals, int to_csc, spg_hcsr* out) {
  return guarded(nullptr, [&] {
    need(out && (nnz == 0 || (rows && cols && vals)), "null argument");
    const int vs = ops_for(sr)->value_size;
    const int64_t nseg = to_csc ? ncols : nrows;
    out->nrows = nrows;
    out->ncols = ncols;
    out->nnz = nnz;
    out->ptr = static_cast<int64_t*>(std::calloc(nseg + 1, sizeof(int64_t)));
    out->idx = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * std::max<int64_t>(nnz, 1)));
    out->vals = std::malloc((size_t)vs * std::max<int64_t>(nnz, 1));
    if (!out->ptr || !out->idx || !out->vals) fail(SPG_ERR_OOM, "host allocation failed");
    const int64_t* seg = to_csc ? cols : rows;
    const int64_t* oth = to_csc ? rows : cols;
    for (int64_t k = 0; k < nnz; ++k) {
      if (rows[k] < 0 || rows[k] >= nrows || cols[k] < 0 || cols[k] >= ncols)
        fail(SPG_ERR_MALFORMED, "coo tuple outside the matrix");
      ++out->ptr[seg[k] + 1];
    }
    for (int64_t s = 0; s < nseg; ++s) out->ptr[s + 1] += out->ptr[s];
    std::vector<int64_t> cur(out->ptr, out->ptr + nseg);
    const char* v = static_cast<const char*>(vals);
    char* ov = static_cast<char*>(out->vals);
    for (int64_t k = 0; k < nnz; ++k) {  // stable counting sort by segment
      const int64_t p = cur[seg[k]]++;
      out->idx[p] = oth[k];
      std::memcpy(ov + (size_t)vs * p, v + (size_t)vs * k, vs);
    }
  });
}

void spg_free(void* p) { host_release(p); }

void spg_block_free(spg_block* b) {
  if (!b) return;
  for (void* p : {(void*)b->csc.ptr, (void*)b->csc.idx, b->csc.vals, (void*)b->dcsc.jc, (void*)b->dcsc.cp,
                  (void*)b->dcsc.rowids, b->dcsc.vals})
    host_release(p);
  std::memset(b, 0, sizeof(*b));
}

int spg_distribute(spg_ctx* c, int sr, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                   const int64_t* cols, const void* vals, int pr, int pc, int only_rank, spg_block* blocks) {
  const int nout = only_rank >= 0 ? 1 : std::max(pr, 0) * std::max(pc, 0);
  if (blocks && pr > 0 && pc > 0) std::memset(blocks, 0, sizeof(spg_block) * (size_t)nout);
  const int rc = guarded(c, [&] {
    need(c && blocks && (nnz == 0 || (rows && cols && vals)), "null argument");
    need(nrows >= 0 && ncols >= 0 && nnz >= 0, "negative dims");
    if (pr < 1 || pc < 1) fail(SPG_ERR_GRID, "distribute: grid must be at least 1 x 1");
    if (only_rank >= pr * pc) fail(SPG_ERR_GRID, "distribute: rank outside the grid");
    if ((nrows + pr - 1) / pr > INT32_MAX || (ncols + pc - 1) / pc > INT32_MAX)
      fail(SPG_ERR_INVALID_RANGE, "block dimension exceeds int32 indices");
    use_device(c);
    distribute_coo(c, ops_for(sr), nrows, ncols, nnz, rows, cols, vals, pr, pc, only_rank, blocks,
                   [](size_t bytes) -> void* {
                     try {
                       return pinned().get(bytes);
                     } catch (...) {
                       return nullptr;
                     }
                   });
  });
  if (rc != SPG_OK && blocks && pr > 0 && pc > 0)
    for (int k = 0; k < nout; ++k) spg_block_free(&blocks[k]);
  return rc;
}

void* spg_host_alloc(uint64_t bytes) {
  try {
    return pinned().get((size_t)bytes);
  } catch (...) {
    return nullptr;
  }
}

int spg_host_register(void* p, uint64_t bytes) {
  return guarded(nullptr, [&] {
    if (!p || bytes == 0) return;
    const cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterPortable);
    if (e != cudaSuccess) cudaGetLastError();  // not sticky: later launches must not see it
    if (e == cudaErrorHostMemoryAlreadyRegistered) return;
    SPG_CUDA(e);
  });
}

int spg_host_unregister(void* p) {
  return guarded(nullptr, [&] {
    if (!p) return;
    const cudaError_t e = cudaHostUnregister(p);
    if (e != cudaSuccess) cudaGetLastError();
    if (e == cudaErrorHostMemoryNotRegistered) return;
    SPG_CUDA(e);
  });
}

void spg_block_range(int64_t n, int q, int idx, int64_t* begin, int64_t* end) {
  // dist_matrix.hpp:23-28: larger ranges first
  const int64_t base = n / q, extra = n % q;
  const int64_t b = idx * base + std::min<int64_t>(idx, extra);
  *begin = b;
  *end = b + base + (idx < extra ? 1 : 0);
}

void spg_round_range(int64_t n, int rounds, int round, int64_t* begin, int64_t* end) {
  // summa.hpp:103-107: first half gets ceil(n/2)
  if (rounds == 1) {
    *begin = 0;
    *end = n;
    return;
  }
  const int64_t mid = (n + 1) / 2;
  *begin = round == 0 ? 0 : mid;
  *end = round == 0 ? mid : n;
}

int spg_summa_schedule(int64_t inner, int pr, int pc, spg_stage* out, int cap) {
  // Square grids: exactly the reference's q stages (summa.hpp:290-306),
  // empty blocks included.  pr x pc grids: the common refinement of A's pc
  // column blocks and B's pr row blocks of the inner dimension (empty
  // intervals dropped), so every stage has one A-panel owner and one
  // B-panel owner.
  if (pr < 1 || pc < 1 || inner < 0) return -SPG_ERR_GRID;
  auto owner = [](int64_t total, int q, int64_t x) {
    // block_index_of (dist_matrix.hpp:31-37)
    const int64_t base = total / q, extra = total % q, wide = extra * (base + 1);
    if (x < wide) return (int)(x / (base + 1));
    return (int)(extra + (x - wide) / base);
  };
  std::vector<spg_stage> st;
  if (pr == pc) {
    for (int s = 0; s < pr; ++s) {
      int64_t b, e;
      spg_block_range(inner, pr, s, &b, &e);
      st.push_back(spg_stage{b, e, s, s, 0, 0});
    }
  } else {
    std::vector<int64_t> cuts{0, inner};
    for (int j = 1; j < pc; ++j) {
      int64_t b, e;
      spg_block_range(inner, pc, j, &b, &e);
      cuts.push_back(b);
    }
    for (int i = 1; i < pr; ++i) {
      int64_t b, e;
      spg_block_range(inner, pr, i, &b, &e);
      cuts.push_back(b);
    }
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    for (size_t k = 0; k + 1 < cuts.size(); ++k) {
      const int64_t lo = cuts[k], hi = cuts[k + 1];
      if (hi <= lo) continue;
      spg_stage s{lo, hi, owner(inner, pc, lo), owner(inner, pr, lo), 0, 0};
      int64_t ab, ae, bb, be;
      spg_block_range(inner, pc, s.a_col_block, &ab, &ae);
      spg_block_range(inner, pr, s.b_row_block, &bb, &be);
      s.a_off = lo - ab;
      s.b_off = lo - bb;
      st.push_back(s);
    }
  }
  for (size_t k = 0; k < st.size() && (int)k < cap && out; ++k) out[k] = st[k];
  return (int)st.size();
}

}  // extern "C"
