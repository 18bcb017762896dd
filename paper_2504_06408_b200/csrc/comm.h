// Node-local communication fabric for the SUMMA broadcasts.
//
// Replaces the reference's simulated FabricEngine (fabric.hpp:76-311) with
// real transports on one 8-GPU box, one process per GPU:
//   * a POSIX shared-memory segment per job holds the rendezvous state:
//     cross-process barriers per scope (grid row / grid column / world), the
//     24-byte size-triple slots of exchange_sizes (fabric.hpp:86-95, always
//     host path), the NCCL unique id, an abort flag, and per-scope pinned
//     staging buffers (cudaHostRegister'ed) for host-path broadcasts;
//   * device-path broadcasts use NCCL (ncclBroadcast on row/column
//     communicators split from a world communicator) over NVLink 5 /
//     NVSwitch, or a P2P pull over CUDA IPC;
//   * the path of each payload is choose_path(bytes, cfg) (comm.hpp:45-55):
//     device iff bytes >= threshold in hybrid mode.
// A failing rank raises the shared abort flag; peers blocked in a barrier
// then throw AbortedError, and a barrier that times out throws
// DeadlockError (fabric.hpp:141-149, :264-290).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <string>

#include "../../include/spgemm_b200.h"

struct spg_comm;

namespace spg {

constexpr int kMaxGridSide = 16;

struct CommCounters {
  uint64_t host_bcasts = 0, device_bcasts = 0, bytes_host = 0, bytes_device = 0, size_exchanges = 0;
  double ms_bcast = 0, ms_copy = 0;
};

// Internal API used by the SUMMA driver (all ranks of a scope must call the
// same sequence; `root` is the scope-local index).
int comm_scope_size(const spg_comm* c, int scope);
int comm_scope_index(const spg_comm* c, int scope);  // my index within the scope
int comm_grid_row(const spg_comm* c);
int comm_grid_col(const spg_comm* c);
int comm_pr(const spg_comm* c);
int comm_pc(const spg_comm* c);
void comm_exchange_sizes(spg_comm* c, int scope, int root, int64_t triple[3]);
// returns SPG_PATH_*; `stream` orders the transfer after prior device work
int comm_bcast(spg_comm* c, int scope, int root, void* buf, uint64_t bytes, int mode, uint64_t threshold,
               cudaStream_t stream, bool device_buffer, bool wait = true);
// after device broadcasts issued with wait = false: drain the stream, check NCCL errors
void comm_bcast_wait(spg_comm* c, cudaStream_t stream);
void comm_barrier(spg_comm* c);
int comm_world_rank(const spg_comm* c);
int comm_world_size(const spg_comm* c);
// every rank contributes n int64 (host), every rank receives world*n (host), over NCCL
void comm_allgather_i64(spg_comm* c, const int64_t* mine, int n, int64_t* all, cudaStream_t stream);
// device buffers to world rank `root` over NCCL (send on non-roots; the root receives
// recv[r] of recv_bytes[r] from every other rank r)
void comm_gather_bytes(spg_comm* c, int root, const void* send, uint64_t bytes, void* const* recv,
                       const uint64_t* recv_bytes, cudaStream_t stream);
void comm_abort(spg_comm* c, const std::string& why);
CommCounters& comm_counters(spg_comm* c);

}  // namespace spg
