// Node-local fabric: shared-memory rendezvous + pinned host staging + NCCL
// (see comm.h for the design and the reference mapping).
#include "comm.h"

#include <fcntl.h>
#include <nccl.h>
#include <sched.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <thread>

#include "common.cuh"

namespace spg {
namespace {

constexpr uint64_t kMagic = 0x53504742323030ULL;  // "SPGB200"

struct alignas(64) Barrier {
  std::atomic<uint32_t> count;
  std::atomic<uint32_t> gen;
  char pad[56];
};

struct alignas(64) Slot {
  int64_t triple[3];
  char pad[40];
};

struct Header {
  std::atomic<uint64_t> magic;
  int32_t world, pr, pc;
  uint64_t staging_bytes;
  std::atomic<int32_t> attached;
  std::atomic<int32_t> abort_flag;
  char abort_msg[256];
  std::atomic<int32_t> uid_ready;
  unsigned char uid[sizeof(ncclUniqueId)];
  Barrier world_bar;
  Barrier scope_bar[2][kMaxGridSide];
  Slot slot[2][kMaxGridSide];
  unsigned char dev_uuid[kMaxGridSide * kMaxGridSide][16];  // per rank: its GPU (cudaDeviceProp::uuid)
};

size_t header_bytes() { return (sizeof(Header) + 4095) & ~size_t(4095); }

double timeout_s() {
  const char* e = std::getenv("SPG_COMM_TIMEOUT_S");
  return e ? std::atof(e) : 600.0;
}

}  // namespace
}  // namespace spg

struct spg_comm {
  std::string name;
  int world = 1, rank = 0, pr = 1, pc = 1, device = -1;
  int row = 0, col = 0;
  spg::Header* hdr = nullptr;
  size_t map_bytes = 0;
  char* staging = nullptr;  // 2 * (pr + pc) scope regions
  uint64_t staging_bytes = 0;
  bool registered = false;
  ncclComm_t world_comm = nullptr, row_comm = nullptr, col_comm = nullptr;
  int transport = SPG_DEV_NCCL;
  bool shared_gpu = false;  // several ranks on one GPU: no NCCL communicator, host path only
  std::string last_error;
  spg::CommCounters counters;
  bool owner = false;
};

namespace spg {
namespace {

void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(SPG_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

void raise_abort(spg_comm* c) {
  fail(SPG_ERR_ABORTED, std::string("peer failure: ") + c->hdr->abort_msg);
}

void barrier_wait(spg_comm* c, Barrier& b, int n) {
  if (n <= 1) return;
  const uint32_t g = b.gen.load(std::memory_order_acquire);
  if (b.count.fetch_add(1, std::memory_order_acq_rel) == (uint32_t)n - 1) {
    b.count.store(0, std::memory_order_relaxed);
    b.gen.fetch_add(1, std::memory_order_release);
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  const double limit = timeout_s();
  uint64_t spins = 0;
  while (b.gen.load(std::memory_order_acquire) == g) {
    if (c->hdr->abort_flag.load(std::memory_order_acquire)) raise_abort(c);
    if (++spins > 2000) {
      sched_yield();
      if ((spins & 1023) == 0) {
        const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > limit) {
          comm_abort(c, "deadlock: barrier timed out after " + std::to_string((int)el) + " s on rank " +
                            std::to_string(c->rank));
          fail(SPG_ERR_DEADLOCK, "deadlock: no collective can complete (barrier timeout)");
        }
      }
    }
  }
}

Barrier& scope_barrier(spg_comm* c, int scope) {
  return c->hdr->scope_bar[scope][scope == SPG_SCOPE_ROW ? c->row : c->col];
}

char* staging_region(spg_comm* c, int scope) {
  const int idx = scope == SPG_SCOPE_ROW ? c->row : c->pr + c->col;
  return c->staging + (size_t)idx * c->staging_bytes;
}

}  // namespace

int comm_scope_size(const spg_comm* c, int scope) { return scope == SPG_SCOPE_ROW ? c->pc : c->pr; }
int comm_scope_index(const spg_comm* c, int scope) { return scope == SPG_SCOPE_ROW ? c->col : c->row; }
int comm_grid_row(const spg_comm* c) { return c->row; }
int comm_grid_col(const spg_comm* c) { return c->col; }
int comm_pr(const spg_comm* c) { return c->pr; }
int comm_pc(const spg_comm* c) { return c->pc; }
CommCounters& comm_counters(spg_comm* c) { return c->counters; }

void comm_abort(spg_comm* c, const std::string& why) {
  if (!c || !c->hdr) return;
  int expected = 0;
  if (c->hdr->abort_flag.compare_exchange_strong(expected, 1)) {
    std::strncpy(c->hdr->abort_msg, why.c_str(), sizeof(c->hdr->abort_msg) - 1);
  }
}

void comm_barrier(spg_comm* c) { barrier_wait(c, c->hdr->world_bar, c->world); }

void comm_bcast_wait(spg_comm* c, cudaStream_t stream) {
  SPG_CUDA(cudaStreamSynchronize(stream));
  for (ncclComm_t comm : {c->row_comm, c->col_comm}) {
    if (!comm) continue;
    ncclResult_t async_err = ncclSuccess;
    nccl_check(ncclCommGetAsyncError(comm, &async_err), "ncclCommGetAsyncError");
    nccl_check(async_err, "ncclBroadcast (async)");
  }
}
int comm_world_rank(const spg_comm* c) { return c->rank; }
int comm_world_size(const spg_comm* c) { return c->world; }

void comm_allgather_i64(spg_comm* c, const int64_t* mine, int n, int64_t* all, cudaStream_t stream) {
  if (!c->world_comm) fail(SPG_ERR_ARG, "allgather needs a GPU communicator");
  int64_t* d = nullptr;
  SPG_CUDA(cudaMallocAsync(&d, sizeof(int64_t) * n * (c->world + 1), stream));
  SPG_CUDA(cudaMemcpyAsync(d, mine, sizeof(int64_t) * n, cudaMemcpyHostToDevice, stream));
  nccl_check(ncclAllGather(d, d + n, n, ncclInt64, c->world_comm, stream), "ncclAllGather");
  SPG_CUDA(cudaMemcpyAsync(all, d + n, sizeof(int64_t) * n * c->world, cudaMemcpyDeviceToHost, stream));
  SPG_CUDA(cudaFreeAsync(d, stream));
  SPG_CUDA(cudaStreamSynchronize(stream));
}

void comm_gather_bytes(spg_comm* c, int root, const void* send, uint64_t bytes, void* const* recv,
                       const uint64_t* recv_bytes, cudaStream_t stream) {
  if (!c->world_comm) fail(SPG_ERR_ARG, "gather needs a GPU communicator");
  if (root < 0 || root >= c->world) fail(SPG_ERR_PROTOCOL, "gather root outside the world");
  nccl_check(ncclGroupStart(), "ncclGroupStart");
  if (c->rank != root) {
    if (bytes) nccl_check(ncclSend(send, bytes, ncclUint8, root, c->world_comm, stream), "ncclSend");
  } else {
    for (int r = 0; r < c->world; ++r)
      if (r != root && recv_bytes[r])
        nccl_check(ncclRecv(recv[r], recv_bytes[r], ncclUint8, r, c->world_comm, stream), "ncclRecv");
  }
  nccl_check(ncclGroupEnd(), "ncclGroupEnd");
  SPG_CUDA(cudaStreamSynchronize(stream));
  ncclResult_t async_err = ncclSuccess;
  nccl_check(ncclCommGetAsyncError(c->world_comm, &async_err), "ncclCommGetAsyncError");
  nccl_check(async_err, "gather (async)");
}

// Rank::exchange_sizes (fabric.hpp:335-338): root publishes, all read.
void comm_exchange_sizes(spg_comm* c, int scope, int root, int64_t triple[3]) {
  const int n = comm_scope_size(c, scope);
  if (root < 0 || root >= n)
    fail(SPG_ERR_PROTOCOL, "broadcast root " + std::to_string(root) + " is outside the scope");
  Slot& s = c->hdr->slot[scope][scope == SPG_SCOPE_ROW ? c->row : c->col];
  const bool me = comm_scope_index(c, scope) == root;
  if (me) std::memcpy(s.triple, triple, sizeof(s.triple));
  barrier_wait(c, scope_barrier(c, scope), n);
  if (!me) std::memcpy(triple, s.triple, sizeof(s.triple));
  barrier_wait(c, scope_barrier(c, scope), n);
  ++c->counters.size_exchanges;
}

int comm_bcast(spg_comm* c, int scope, int root, void* buf, uint64_t bytes, int mode, uint64_t threshold,
               cudaStream_t stream, bool device_buffer, bool wait) {
  const int n = comm_scope_size(c, scope);
  if (root < 0 || root >= n)
    fail(SPG_ERR_PROTOCOL, "broadcast root " + std::to_string(root) + " is outside the scope");
  // choose_path (comm.hpp:45-55)
  int path;
  if (mode == SPG_COMM_HOST_ONLY) path = SPG_PATH_HOST;
  else if (mode == SPG_COMM_DEVICE_ONLY) path = SPG_PATH_DEVICE;
  else path = bytes >= threshold ? SPG_PATH_DEVICE : SPG_PATH_HOST;
  if (!device_buffer) path = SPG_PATH_HOST;  // host buffers (CPU tests) only travel through shm
  if (path == SPG_PATH_DEVICE && !c->world_comm)
    fail(SPG_ERR_ARG, c->shared_gpu ? "device path unavailable: ranks of this job share a GPU (NCCL needs one GPU "
                                      "per rank); use the host path (SPG_COMM_HOST_ONLY)"
                                    : "device path needs a GPU communicator");
  if (path == SPG_PATH_HOST) {
    ++c->counters.host_bcasts;
    c->counters.bytes_host += bytes;
  } else {
    ++c->counters.device_bcasts;
    c->counters.bytes_device += bytes;
  }
  if (n <= 1 || bytes == 0) return path;
  const auto t0 = std::chrono::steady_clock::now();
  const bool me = comm_scope_index(c, scope) == root;
  if (path == SPG_PATH_DEVICE) {
    ncclComm_t comm = scope == SPG_SCOPE_ROW ? c->row_comm : c->col_comm;
    nccl_check(ncclBroadcast(buf, buf, bytes, ncclUint8, root, comm, stream), "ncclBroadcast");
    if (wait) {
      SPG_CUDA(cudaStreamSynchronize(stream));
      ncclResult_t async_err = ncclSuccess;
      nccl_check(ncclCommGetAsyncError(comm, &async_err), "ncclCommGetAsyncError");
      nccl_check(async_err, "ncclBroadcast (async)");
    }
  } else {
    // Root D2H into pinned shm staging, receivers H2D; two half-slots
    // pipeline consecutive chunks (root fills chunk i+1 while peers drain i).
    char* stage = staging_region(c, scope);
    const uint64_t half = c->staging_bytes / 2;
    Barrier& bar = scope_barrier(c, scope);
    char* p = static_cast<char*>(buf);
    uint64_t i = 0;
    double copy_ms = 0;
    for (uint64_t off = 0; off < bytes; off += half, ++i) {
      const uint64_t len = std::min<uint64_t>(half, bytes - off);
      char* slot = stage + (i & 1) * half;
      const auto c0 = std::chrono::steady_clock::now();
      if (me) {
        if (device_buffer) {
          SPG_CUDA(cudaMemcpyAsync(slot, p + off, len, cudaMemcpyDeviceToHost, stream));
          SPG_CUDA(cudaStreamSynchronize(stream));
        } else {
          std::memcpy(slot, p + off, len);
        }
      }
      copy_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c0).count();
      barrier_wait(c, bar, n);
      const auto c1 = std::chrono::steady_clock::now();
      if (!me) {
        if (device_buffer) {
          SPG_CUDA(cudaMemcpyAsync(p + off, slot, len, cudaMemcpyHostToDevice, stream));
          SPG_CUDA(cudaStreamSynchronize(stream));
        } else {
          std::memcpy(p + off, slot, len);
        }
      }
      copy_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c1).count();
    }
    barrier_wait(c, bar, n);  // staging is free for the next broadcast
    c->counters.ms_copy += copy_ms;
  }
  c->counters.ms_bcast += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return path;
}

void note_host_procs(int n);  // capi.cu: host-side download policy

}  // namespace spg

using namespace spg;

namespace {
thread_local std::string g_comm_err;

template <class F>
int cguard(spg_comm* c, F&& f) {
  try {
    f();
    return SPG_OK;
  } catch (const Error& e) {
    g_comm_err = e.what();
    if (c) {
      c->last_error = e.what();
      if (e.status != SPG_ERR_ABORTED && e.status != SPG_ERR_DEADLOCK) comm_abort(c, e.what());
    }
    return e.status;
  } catch (const std::exception& e) {
    g_comm_err = e.what();
    if (c) {
      c->last_error = e.what();
      comm_abort(c, e.what());
    }
    return SPG_ERR_INTERNAL;
  }
}
}  // namespace

extern "C" {

int spg_comm_create(const char* job, int world, int rank, int pr, int pc, int device, uint64_t staging_bytes,
                    spg_comm** out) {
  spg_comm* c = nullptr;
  const int rc = cguard(nullptr, [&] {
    if (!job || !out) fail(SPG_ERR_ARG, "null argument");
    if (pr < 1 || pc < 1 || pr * pc != world || pr > kMaxGridSide || pc > kMaxGridSide)
      fail(SPG_ERR_GRID, "grid " + std::to_string(pr) + "x" + std::to_string(pc) + " does not hold " +
                             std::to_string(world) + " ranks");
    if (rank < 0 || rank >= world) fail(SPG_ERR_GRID, "rank outside the grid");
    c = new spg_comm();
    spg::note_host_procs(world);  // one node: every rank of the job is on this host
    c->name = std::string("/spg_") + job;
    c->world = world;
    c->rank = rank;
    c->pr = pr;
    c->pc = pc;
    c->row = rank / pc;
    c->col = rank % pc;
    c->device = device;
    c->staging_bytes = staging_bytes ? ((staging_bytes + 8191) & ~uint64_t(8191)) : (uint64_t(32) << 20);
    const size_t total = header_bytes() + (size_t)(pr + pc) * c->staging_bytes;
    c->map_bytes = total;
    int fd = -1;
    if (rank == 0) {
      shm_unlink(c->name.c_str());
      fd = shm_open(c->name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd < 0) fail(SPG_ERR_PROTOCOL, "shm_open(create) failed for " + c->name);
      if (ftruncate(fd, (off_t)total) != 0) {
        close(fd);
        fail(SPG_ERR_OOM, "ftruncate of the shared segment failed (is /dev/shm large enough?)");
      }
      c->owner = true;
    } else {
      const auto t0 = std::chrono::steady_clock::now();
      for (;;) {
        fd = shm_open(c->name.c_str(), O_RDWR, 0600);
        if (fd >= 0) {
          struct stat st;
          if (fstat(fd, &st) == 0 && (size_t)st.st_size >= total) break;
          close(fd);
          fd = -1;
        }
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s())
          fail(SPG_ERR_DEADLOCK, "timed out waiting for rank 0 to create " + c->name);
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
      }
    }
    void* p = mmap(nullptr, total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) fail(SPG_ERR_OOM, "mmap of the shared segment failed");
    c->hdr = static_cast<Header*>(p);
    c->staging = static_cast<char*>(p) + header_bytes();
    if (rank == 0) {
      Header* h = c->hdr;
      h->world = world;
      h->pr = pr;
      h->pc = pc;
      h->staging_bytes = c->staging_bytes;
      h->attached.store(0);
      h->abort_flag.store(0);
      h->uid_ready.store(0);
      if (device >= 0) {
        ncclUniqueId id;
        nccl_check(ncclGetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(h->uid, &id, sizeof(id));
        h->uid_ready.store(1, std::memory_order_release);
      }
      h->magic.store(kMagic, std::memory_order_release);
    } else {
      const auto t0 = std::chrono::steady_clock::now();
      while (c->hdr->magic.load(std::memory_order_acquire) != kMagic) {
        if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s())
          fail(SPG_ERR_DEADLOCK, "timed out waiting for the shared segment header");
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
      }
      if (c->hdr->world != world || c->hdr->pr != pr || c->hdr->pc != pc)
        fail(SPG_ERR_PROTOCOL, "ranks disagree on the grid shape");
    }
    c->hdr->attached.fetch_add(1);
    if (device >= 0) {
      SPG_CUDA(cudaSetDevice(device));
      SPG_CUDA(cudaHostRegister(c->staging, (size_t)(pr + pc) * c->staging_bytes, cudaHostRegisterDefault));
      c->registered = true;
      // ranks sharing a GPU (e.g. a 2x2 grid exercised on a 1-GPU box) cannot
      // form an NCCL communicator: they run with the host path only
      cudaDeviceProp prop{};
      SPG_CUDA(cudaGetDeviceProperties(&prop, device));
      std::memcpy(c->hdr->dev_uuid[rank], &prop.uuid, 16);
      comm_barrier(c);
      for (int r = 0; r < world; ++r)
        if (r != rank && std::memcmp(c->hdr->dev_uuid[r], c->hdr->dev_uuid[rank], 16) == 0) c->shared_gpu = true;
    }
    if (device >= 0 && !c->shared_gpu) {
      while (c->hdr->uid_ready.load(std::memory_order_acquire) != 1) std::this_thread::sleep_for(std::chrono::milliseconds(1));
      ncclUniqueId id;
      std::memcpy(&id, c->hdr->uid, sizeof(id));
      // NCCL may print its version banner on stdout; keep stdout clean for
      // callers that emit machine-readable output (bench.py's JSON line).
      std::fflush(stdout);
      const int saved = dup(1);
      if (saved >= 0) dup2(2, 1);
      struct Restore {
        int fd;
        ~Restore() {
          if (fd >= 0) {
            std::fflush(stdout);
            dup2(fd, 1);
            close(fd);
          }
        }
      } restore{saved};
      nccl_check(ncclCommInitRank(&c->world_comm, world, id, rank), "ncclCommInitRank");
      nccl_check(ncclCommSplit(c->world_comm, c->row, c->col, &c->row_comm, nullptr), "ncclCommSplit(row)");
      nccl_check(ncclCommSplit(c->world_comm, c->col, c->row, &c->col_comm, nullptr), "ncclCommSplit(col)");
    }
    comm_barrier(c);
    if (rank == 0) shm_unlink(c->name.c_str());  // everyone is attached; the mapping stays valid
    *out = c;
  });
  if (rc != SPG_OK && c) {
    if (c->hdr) munmap(c->hdr, c->map_bytes);
    delete c;
  }
  return rc;
}

void spg_comm_destroy(spg_comm* c) {
  if (!c) return;
  if (c->row_comm) ncclCommDestroy(c->row_comm);
  if (c->col_comm) ncclCommDestroy(c->col_comm);
  if (c->world_comm) ncclCommDestroy(c->world_comm);
  if (c->registered) cudaHostUnregister(c->staging);
  if (c->hdr) munmap(c->hdr, c->map_bytes);
  delete c;
}

const char* spg_comm_last_error(const spg_comm* c) { return c ? c->last_error.c_str() : g_comm_err.c_str(); }

int spg_comm_barrier(spg_comm* c) {
  return cguard(c, [&] { comm_barrier(c); });
}

int spg_exchange_sizes(spg_comm* c, int scope, int root, int64_t triple[3]) {
  return cguard(c, [&] { comm_exchange_sizes(c, scope, root, triple); });
}

int spg_bcast(spg_comm* c, int scope, int root, void* buf, uint64_t bytes, int mode, uint64_t threshold,
              int* path_out) {
  return cguard(c, [&] {
    cudaPointerAttributes attr{};
    bool dev = false;
    if (c->device >= 0 && cudaPointerGetAttributes(&attr, buf) == cudaSuccess)
      dev = attr.type == cudaMemoryTypeDevice;
    cudaGetLastError();
    cudaStream_t s = nullptr;
    const int p = comm_bcast(c, scope, root, buf, bytes, mode, threshold, s, dev);
    if (path_out) *path_out = p;
  });
}

int spg_comm_set_device_transport(spg_comm* c, int transport) {
  return cguard(c, [&] {
    if (transport == SPG_DEV_P2P)
      fail(SPG_ERR_ARG, "device transport P2P is not implemented; the device path uses NCCL over NVLink");
    if (transport != SPG_DEV_NCCL) fail(SPG_ERR_ARG, "unknown transport");
    c->transport = transport;
  });
}

int spg_comm_has_device_path(const spg_comm* c) { return c && c->world_comm ? 1 : 0; }

}  // extern "C"
