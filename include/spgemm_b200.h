/*
 * spgemm_b200.h — C-ABI of the B200-native distributed semiring SpGEMM engine.
 *
 * This is the drop-in boundary for the reference library `spsumma`
 * (/root/reference/proj/include/spsumma, header-only C++20).  Each entry point
 * below names the reference interface it replaces (file:line relative to that
 * directory).  Plain pointers and sizes only: no C++ or torch types cross it.
 * The reference-shaped C++ facade in include/spsumma_b200.hpp sits on top.
 *
 * Conventions
 *  - Semirings are identified by SPG_SR_* ids (the reference's closed
 *    SemiringId table, semiring.hpp:122-149, plus the two BASELINE semirings).
 *  - Host matrices (spg_hcsr) use the reference's index width: int64 offsets
 *    and int64 indices (common.hpp:10), values in ValueCodec byte layout
 *    (serialize.hpp:29-76; bool = 1 byte 0/1).
 *  - Device matrices (spg_dcsr) use int64 offsets and int32 block-local
 *    indices; values have the same byte layout as on the host.
 *  - A CSR and a CSC share the struct: `ptr` runs over rows (CSR) or columns
 *    (CSC); nrows/ncols are always the logical dims.
 *  - Every call returns an spg_status; the message of the last failure is in
 *    spg_last_error(ctx) (or spg_last_error(NULL) for calls without a ctx).
 *    Status codes map 1:1 onto the reference exception classes
 *    (common.hpp:12-73) so the C++ facade rethrows the matching type.
 */
#ifndef SPGEMM_B200_H
#define SPGEMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPG_API __attribute__((visibility("default")))

/* semiring ids: 0-3 are the reference built-ins (semiring.hpp:43-120) */
enum {
  SPG_SR_ARITHMETIC = 0,   /* double (+, x)                       semiring.hpp:43-54 */
  SPG_SR_MINPLUS = 1,      /* double (min, +), zero = +inf         semiring.hpp:59-72 */
  SPG_SR_BOOLEAN = 2,      /* bool (or, and), 1 byte               semiring.hpp:75-86 */
  SPG_SR_MINSELECT = 3,    /* {double, int64}, non-commutative mul semiring.hpp:97-120 */
  SPG_SR_TROPICAL_I32 = 4, /* int32 (min, saturating +)            BASELINE config 2 */
  SPG_SR_MAXTIMES = 5,     /* {double w, uint64 tag} (max, x)      BASELINE config 5 */
  SPG_SR_COUNT = 6
};

/* status codes (reference exception classes, common.hpp:12-73) */
enum {
  SPG_OK = 0,
  SPG_ERR_SHAPE = 1,                 /* ShapeError */
  SPG_ERR_GRID = 2,                  /* GridError */
  SPG_ERR_UNSUPPORTED_SEMIRING = 3,  /* UnsupportedSemiringError */
  SPG_ERR_PROTOCOL = 4,              /* ProtocolError */
  SPG_ERR_MALFORMED = 5,             /* MalformedInputError */
  SPG_ERR_INVALID_RANGE = 6,         /* InvalidRangeError */
  SPG_ERR_INTERNAL = 7,              /* InternalError */
  SPG_ERR_ABORTED = 8,               /* AbortedError */
  SPG_ERR_DEADLOCK = 9,              /* DeadlockError */
  SPG_ERR_CUDA = 10,                 /* CUDA runtime failure */
  SPG_ERR_OOM = 11,                  /* device or host allocation failure */
  SPG_ERR_NCCL = 12,                 /* NCCL failure (surfaces as ProtocolError) */
  SPG_ERR_ARG = 13,                  /* invalid argument (null pointer, bad id) */
  SPG_ERR_UNSUPPORTED_FORMAT = 14    /* UnsupportedFormatError */
};

/* communication paths / modes (comm.hpp:14-55) */
enum { SPG_PATH_HOST = 0, SPG_PATH_DEVICE = 1 };
enum { SPG_COMM_HOST_ONLY = 0, SPG_COMM_DEVICE_ONLY = 1, SPG_COMM_HYBRID = 2 };
/* device transport for the device path */
enum { SPG_DEV_NCCL = 0, SPG_DEV_P2P = 1 };
/* scopes (fabric.hpp:34-43) */
enum { SPG_SCOPE_ROW = 0, SPG_SCOPE_COL = 1 };

typedef struct spg_ctx spg_ctx;
typedef struct spg_comm spg_comm;

/* host CSR/CSC in the reference layout (formats.hpp:39-86) */
typedef struct {
  int64_t nrows, ncols, nnz;
  int64_t* ptr; /* nseg + 1 */
  int64_t* idx; /* nnz */
  void* vals;   /* nnz * spg_value_size(sr) bytes */
} spg_hcsr;

/* host DCSC (formats.hpp:56-70): jc[njc] nonempty column ids, cp[njc + 1] */
typedef struct {
  int64_t nrows, ncols, nnz, njc;
  int64_t* jc;
  int64_t* cp;
  int64_t* rowids;
  void* vals;
} spg_hdcsc;

/* device CSR/CSC */
typedef struct {
  int64_t nrows, ncols, nnz;
  int64_t* ptr; /* device, nseg + 1 */
  int32_t* idx; /* device, nnz */
  void* vals;   /* device, nnz * value size */
} spg_dcsr;

/* per-call statistics of a local multiply / merge */
typedef struct {
  int64_t products;        /* F: intermediate products (flops = 2F) */
  int64_t nnz_out;
  int64_t rows_per_bin[12]; /* 0 empty, 1 warp-ESC, 2 block-ESC, 3/4/5 hash 4K/8K/2K, 6 dense panels,
                               7 hash max, 8 bit-rank (presence bitmap + ranked accumulator),
                               9 rank panels (bit-rank with accumulator panels in rank space),
                               10 bitmap-rank (symbolic bitmap + ranked fold, written straight into C),
                               11 wide rows (too wide for dense panels, too many outputs for a
                                  shared-memory hash: products sorted in HBM, then folded) */
  double ms_analyse;       /* row products + binning + offsets */
  double ms_numeric;       /* accumulate kernels */
  double ms_compact;       /* output scan + compaction */
  double ms_total;
  int64_t kernels;         /* kernels launched by the call */
  int64_t output_mode;     /* 0: U-slot scratch + compaction, 1: exact claims + compaction,
                              2: two passes (count, then write into C),
                              3: bitmap-rank (long rows straight into C, short rows compacted),
                              4: pattern-only (Boolean: column-only count + emit passes) */
  /* bitmap-rank pipeline (output_mode 3): the two phases of the long rows */
  double ms_symbolic;      /* symbolic bitmaps (|| the short rows' kernels) + rowptr scan */
  double ms_fold;          /* rank-space fold into C (|| the short rows' compaction) */
  int64_t bitmap_bytes;    /* bitmap words streamed out by the symbolic pass and back in by the fold */
  int64_t fold_items;      /* (row, rank window) work items of the fold */
} spg_mult_stats;

/* ---------------------------------------------------------------- misc */
SPG_API const char* spg_version(void);
SPG_API const char* spg_last_error(const spg_ctx* ctx); /* ctx may be NULL */
SPG_API int spg_value_size(int sr);
SPG_API int spg_semiring_by_name(const char* name); /* semiring_by_name, semiring.hpp:125-133; -1 if unknown */
SPG_API const char* spg_semiring_name(int sr);
SPG_API int spg_semiring_is_commutative(int sr);  /* SR::is_commutative_mul */
/* User-defined semirings (the reference's SemiringLike plug-in,
   semiring.hpp:28-40, + ValueCodec<T>, serialize.hpp:29-76): a struct with
   value_type, add, mul, zero, one, is_zero, from_real, name,
   is_commutative_mul (all __host__ __device__; optional acc_shared /
   acc_global atomics, small / mul_small fast multiply, add_can_cancel),
   instantiated in the user's own .cu with
       SPG_INSTANTIATE(MySemiring, my_semiring_ops)   (csrc/instantiate.cuh)
   and compiled into the user's shared library.  Registering the table
   returns the id every entry point below accepts as `sr` (values travel as
   their raw little-endian bytes, value_type size 1/2/4/8/16).  Registering
   the same table again returns the same id; names must be unique. */
typedef struct spg_semiring_ops spg_semiring_ops;
SPG_API int spg_register_semiring(const spg_semiring_ops* ops, int* id);

/* ------------------------------------------------------------- context */
SPG_API int spg_device_count(void); /* visible CUDA devices (0 without a GPU) */
SPG_API int spg_ctx_create(int device, spg_ctx** out);
SPG_API void spg_ctx_destroy(spg_ctx* ctx);
SPG_API void* spg_ctx_stream(spg_ctx* ctx);                 /* cudaStream_t */
SPG_API int spg_ctx_set_stream(spg_ctx* ctx, void* stream); /* borrow a caller stream */
SPG_API int spg_ctx_sync(spg_ctx* ctx);
SPG_API uint64_t spg_ctx_kernel_launches(const spg_ctx* ctx);
/* bytes of device scratch the single-pass numeric may use (0 = auto: 45% of free
 * HBM); above it the multiply switches to the exact two-pass mode */
SPG_API int spg_ctx_set_scratch_budget(spg_ctx* ctx, uint64_t bytes);
/* Local-multiply pipeline: SPG_PIPE_AUTO (default) sends rows with more than
   2048 products through the bitmap-rank kernels (symbolic bitmap pass, exact
   rowptr, values folded in rank space straight into C) whenever the output
   width fits a shared-memory bitmap; SPG_PIPE_BINS forces the per-bin
   accumulators (hash / dense panels / bit-rank) with scratch + compaction;
   SPG_PIPE_SORTED is SPG_PIPE_BINS with every dense-panel row sent to the
   sort fallback (products sorted in HBM, then folded) that otherwise serves
   only outputs too wide for dense panels. */
#define SPG_PIPE_AUTO 0
#define SPG_PIPE_BINS 1
#define SPG_PIPE_SORTED 2
SPG_API int spg_ctx_set_pipeline(spg_ctx* ctx, int mode);

/* ---------------------------------------------------- device matrices */
SPG_API int spg_dcsr_alloc(spg_ctx* ctx, int sr, int64_t nrows, int64_t ncols, int64_t nseg,
                           int64_t nnz, spg_dcsr* out);
SPG_API int spg_dcsr_free(spg_ctx* ctx, spg_dcsr* m);
/* rows [row_begin, row_end) of A (x) B — the row-batched form of
   spg_local_multiply (stream C out of HBM batch by batch: multiply a row range,
   consume it — download / checksum — free it, next range) */
SPG_API int spg_local_multiply_rows(spg_ctx* ctx, int sr, const spg_dcsr* a, const spg_dcsr* b,
                                    int64_t row_begin, int64_t row_end, spg_dcsr* c, spg_mult_stats* stats);
/* stream-ordered device -> host copy of `bytes` (synchronous on return) */
SPG_API int spg_copy_to_host(spg_ctx* ctx, void* dst, const void* src, uint64_t bytes);
/* H2D of a host CSR (or CSC) with int64 -> int32 index narrowing on device */
SPG_API int spg_upload(spg_ctx* ctx, int sr, const spg_hcsr* h, int is_csc, spg_dcsr* out);
/* D2H into library-allocated host arrays (pinned, recycled by the library:
 * release with spg_hcsr_free, or each array with spg_free) */
SPG_API int spg_download(spg_ctx* ctx, int sr, const spg_dcsr* d, int is_csc, spg_hcsr* out);
SPG_API void spg_hcsr_free(spg_hcsr* h);

/* --------------------------------------------------- hot path (device) */
/* C = A (x) B over sr.  Replaces esc_multiply (local_spgemm.hpp:83-156);
 * same result contract: products mul(a_ik, b_kj), folded per (i, j), zeros
 * dropped, columns strictly increasing.  ShapeError when a.ncols != b.nrows. */
SPG_API int spg_local_multiply(spg_ctx* ctx, int sr, const spg_dcsr* a, const spg_dcsr* b,
                               spg_dcsr* c, spg_mult_stats* stats);

/* Merges C^T partials (CSR, dims block_cols x block_rows each) into the CSC
 * C block.  Replaces merge_partials (summa.hpp:122-172): folds with SR::add,
 * drops zeros; InternalError on an extents mismatch.  `stages`/`rounds`
 * order the fold (stage-major, round-minor) and may be NULL (list order). */
SPG_API int spg_merge_partials(spg_ctx* ctx, int sr, int nparts, const spg_dcsr* parts,
                               const int* stages, const int* rounds, int64_t block_rows,
                               int64_t block_cols, spg_dcsr* c_csc, spg_mult_stats* stats);

/* matrix_checksum (checksum.hpp:20-38) of a device CSR (is_csc = 0) or CSC. */
SPG_API int spg_checksum(spg_ctx* ctx, int sr, const spg_dcsr* m, int is_csc, uint64_t* out);

/* Sum of the per-tuple checksum terms (no dims seed) with every tuple's
 * coordinates shifted by (row_off, col_off): the block-local part of the
 * checksum of a distributed matrix, so ranks' parts add up to the global
 * matrix_checksum (checksum.hpp:20-38 is order-free). */
SPG_API int spg_checksum_part(spg_ctx* ctx, int sr, const spg_dcsr* m, int is_csc, int64_t row_off,
                              int64_t col_off, uint64_t* out);
/* splitmix64(nrows * 31 + ncols): the dims seed of matrix_checksum. */
SPG_API uint64_t spg_checksum_seed(int64_t nrows, int64_t ncols);

/* csr_row_slice / csr_col_slice (summa.hpp:57-98) on device. */
SPG_API int spg_csr_slice(spg_ctx* ctx, int sr, const spg_dcsr* m, int by_rows, int64_t begin,
                          int64_t end, spg_dcsr* out);

/* prepare_block (summa.hpp:30-53): host CSC (dcsc == NULL) or DCSC block ->
 * device CSR of the block's transpose (dcsc_decompress on device, then the
 * zero-copy reinterpretation).  UnsupportedSemiringError for minselect. */
SPG_API int spg_prepare_block(spg_ctx* ctx, int sr, const spg_hcsr* csc, const spg_hdcsc* dcsc,
                              spg_dcsr* prepared);

/* ------------------------------------- reference-shaped host drop-ins */
/* esc_multiply on host CSR operands (local_spgemm.hpp:83-85): H2D, device
 * multiply, D2H.  The output arrays are library-allocated (spg_hcsr_free). */
SPG_API int spg_esc_multiply(spg_ctx* ctx, int sr, const spg_hcsr* a, const spg_hcsr* b,
                             spg_hcsr* c, spg_mult_stats* stats);

/* generate_rmat<SR>(scale, edge_factor, seed) (rmat.hpp:15-60), bit-identical
 * tuples, normalised row-major.  Returns host COO arrays (free with spg_free). */
SPG_API int spg_generate_rmat(int sr, int scale, double edge_factor, uint64_t seed,
                              int64_t* nrows, int64_t* nnz, int64_t** rows, int64_t** cols,
                              void** vals);
/* Erdos-Renyi-style generator with `d` column draws per row (counter-based,
 * deduplicated) and a 3D 27-point stencil Laplacian
 * (config 4).  value_mode 0: from_real(0.5 + u01); 1: maxtimes {0.5+u01, hash}. */
SPG_API int spg_generate_er(int sr, int64_t n, int d, uint64_t seed, int value_mode,
                            int64_t* nnz, int64_t** rows, int64_t** cols, void** vals);
SPG_API int spg_generate_stencil27(int sr, int64_t N, int64_t* nrows, int64_t* nnz,
                                   int64_t** rows, int64_t** cols, void** vals);
/* The same generators restricted to the block rows [r0, r1) x cols [c0, c1)
 * (global indices), so each rank of a grid builds only its own block. */
SPG_API int spg_generate_er_block(int sr, int64_t n, int d, uint64_t seed, int value_mode, int64_t r0,
                                  int64_t r1, int64_t c0, int64_t c1, int64_t* nnz, int64_t** rows,
                                  int64_t** cols, void** vals);
SPG_API int spg_generate_stencil27_block(int sr, int64_t N, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                                         int64_t* nrows, int64_t* nnz, int64_t** rows, int64_t** cols,
                                         void** vals);
/* read_matrix_market<SR>(path) (matrix_market.hpp:43-141): ASCII coordinate
 * file (real / integer / pattern, general / symmetric) -> normalised COO
 * (normalize_coo, formats.hpp:105-133).  MalformedInputError "path:line: what"
 * for structural errors, UnsupportedFormatError for other headers.  Host
 * arrays freed with spg_free. */
SPG_API int spg_read_matrix_market(int sr, const char* path, int64_t* nrows, int64_t* ncols, int64_t* nnz,
                                   int64_t** rows, int64_t** cols, void** vals);
/* normalised COO (row-major, unique) -> CSR / CSC host arrays, no copies of
 * the reference's fold semantics needed (input already unique). */
SPG_API int spg_coo_to_csr(int sr, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                           const int64_t* cols, const void* vals, int to_csc, spg_hcsr* out);
SPG_API void spg_free(void* p); /* any host array returned by the library */
/* Page-locked host memory from the library's caching allocator (plain
 * malloc when the driver refuses); release with spg_free.  NULL on OOM. */
SPG_API void* spg_host_alloc(uint64_t bytes);
/* Page-lock (pin) / unpin caller-owned host memory so uploads run at full
 * PCIe speed (cudaHostRegister; the caller keeps ownership). */
SPG_API int spg_host_register(void* p, uint64_t bytes);
SPG_API int spg_host_unregister(void* p);

/* ------------------------------------------------ distributed (SUMMA) */
/* Grid helpers: block_range (dist_matrix.hpp:23-28), round_range
 * (summa.hpp:103-107), and the pr x pc stage schedule (common refinement of
 * A's column blocks and B's row blocks; equals the reference's q stages for
 * a square grid).  Pure host functions, usable without a GPU. */
SPG_API void spg_block_range(int64_t n, int q, int idx, int64_t* begin, int64_t* end);
SPG_API void spg_round_range(int64_t n, int rounds, int round, int64_t* begin, int64_t* end);
typedef struct {
  int64_t lo, hi;    /* global inner-dimension interval */
  int a_col_block;   /* A panel root column (grid col) */
  int b_row_block;   /* B panel root row (grid row) */
  int64_t a_off;     /* interval start relative to A's column block */
  int64_t b_off;     /* interval start relative to B's row block */
} spg_stage;
SPG_API int spg_summa_schedule(int64_t inner, int pr, int pc, spg_stage* out, int cap);

/* One process per GPU.  `job` names the shared-memory rendezvous segment
 * (same on every rank of a job); rank = grid_row * pc + grid_col. */
SPG_API int spg_comm_create(const char* job, int world, int rank, int pr, int pc, int device,
                            uint64_t staging_bytes, spg_comm** out);
SPG_API void spg_comm_destroy(spg_comm* comm);
SPG_API const char* spg_comm_last_error(const spg_comm* comm);
SPG_API int spg_comm_barrier(spg_comm* comm);
/* Rank::exchange_sizes (fabric.hpp:335-338): host path always. */
SPG_API int spg_exchange_sizes(spg_comm* comm, int scope, int root, int64_t triple[3]);
/* Rank::bcast (fabric.hpp:343-349) of a device buffer; path chosen by
 * choose_path(bytes, {mode, threshold}) (comm.hpp:45-55).  *path_out gets
 * SPG_PATH_HOST or SPG_PATH_DEVICE.  `root` is the scope-local index. */
SPG_API int spg_bcast(spg_comm* comm, int scope, int root, void* dev_buf, uint64_t bytes,
                      int mode, uint64_t threshold, int* path_out);
SPG_API int spg_comm_set_device_transport(spg_comm* comm, int transport); /* SPG_DEV_NCCL (P2P: SPG_ERR_ARG, not implemented) */
/* 1 when the device path is available (one GPU per rank: NCCL row/column
   communicators); 0 when ranks share a GPU, which runs the host path only */
SPG_API int spg_comm_has_device_path(const spg_comm* comm);

typedef struct {
  int two_round;      /* SummaOptions::two_round (summa.hpp:174-177) */
  int comm_mode;      /* CommConfig::mode (comm.hpp:36-39) */
  uint64_t threshold; /* CommConfig::threshold_bytes */
  uint64_t threshold_col; /* threshold for the grid-column scope (fanout pr); 0 = same as threshold
                             (which then applies to both scopes; the row scope has fanout pc) */
  int fuse_stages;    /* 1: keep every received panel and run ONE fused local multiply over the
                         concatenated panels (no partials, no merge; fold order = ascending k);
                         0: the reference's per-stage multiplies + merge_partials */
  int output;         /* SPG_SUMMA_OUT_BLOCK (0): this rank's C block in HBM;
                         SPG_SUMMA_OUT_CHECKSUM (1): C larger than HBM — the fused multiply runs
                         in column batches of the block (<= batch_bytes of C each), every batch
                         is checksummed (matrix_checksum terms, checksum.hpp:20-38) and
                         released; the ledger carries the block's checksum share and nnz and
                         the returned block is empty */
  uint64_t batch_bytes; /* batch size bound for output = 1 (0: 40% of free device memory) */
} spg_summa_opts;
#define SPG_SUMMA_OUT_BLOCK 0
#define SPG_SUMMA_OUT_CHECKSUM 1

/* CostLedger (cost_ledger.hpp:31-56) with measured instead of modelled time. */
typedef struct {
  double ms[5]; /* prepare, broadcast, local_multiply, merge, copy */
  uint64_t host_bcasts, device_bcasts, bytes_host_path, bytes_device_path;
  uint64_t size_exchanges, local_multiply_calls, skipped_stages, peak_bcast_buffer_bytes;
  int64_t products; /* F over this rank's local multiplies */
  double ms_total;  /* time-to-C on this rank */
  /* collectives this rank ROOTED: the reference's ledger charges each
     collective instance once (fabric.hpp:220-241), so summing these over
     the ranks reproduces its host/device broadcast and size-exchange counts */
  uint64_t rooted_host_bcasts, rooted_device_bcasts, rooted_size_exchanges;
  uint64_t checksum_part; /* output = SPG_SUMMA_OUT_CHECKSUM: this block's matrix_checksum terms */
  int64_t nnz_out;        /* nnz of this rank's C block (both output modes) */
  int64_t batches;        /* column batches of the streamed multiply (1 when materialised) */
  int64_t left_nnz;       /* entries of the fused multiply's left operand (received B panels) */
} spg_ledger;

/* summa25_multiply (summa.hpp:248-349), one rank's program.  a_block /
 * b_block are this rank's host blocks as CSC, or DCSC when the dcsc pointer
 * is non-NULL (LocalBlock, dist_matrix.hpp:41-53).  a_nrows.. are the global
 * dims.  Output: this rank's C block as device CSC (block_rows x block_cols). */
SPG_API int spg_summa25_multiply(spg_comm* comm, spg_ctx* ctx, int sr, int64_t a_nrows,
                                 int64_t a_ncols, int64_t b_ncols, const spg_hcsr* a_csc,
                                 const spg_hdcsc* a_dcsc, const spg_hcsr* b_csc,
                                 const spg_hdcsc* b_dcsc, const spg_summa_opts* opts,
                                 spg_dcsr* c_csc, spg_ledger* ledger);

/* One rank's block as distribute builds it (LocalBlock, dist_matrix.hpp:41-53):
 * global extents [row_begin, row_end) x [col_begin, col_end) and storage CSC
 * (is_dcsc == 0, `csc`) or DCSC (is_dcsc == 1, `dcsc`); host arrays owned by
 * the library (spg_block_free). */
typedef struct {
  int64_t row_begin, row_end, col_begin, col_end;
  int is_dcsc;
  spg_hcsr csc;
  spg_hdcsc dcsc;
} spg_block;

/* distribute (dist_matrix.hpp:69-111) ON THE GPU: the host COO (global
 * indices, any order, duplicates allowed) is uploaded once, every tuple is
 * routed to the block owning it (block_index_of, dist_matrix.hpp:31-37) on a
 * pr x pc grid (rank = i * pc + j), each block is built as coo_to_csc does
 * (formats.hpp:138-180: stable column-major order, duplicates folded with
 * SR::add in input order, zeros dropped) by one device radix sort, and a block
 * with fewer than half of its columns populated is stored DCSC.  only_rank < 0
 * builds all pr * pc blocks into blocks[rank]; only_rank >= 0 builds that
 * rank's block alone into blocks[0] (one process per GPU).
 * MalformedInputError for a tuple outside nrows x ncols. */
SPG_API int spg_distribute(spg_ctx* ctx, int sr, int64_t nrows, int64_t ncols, int64_t nnz,
                           const int64_t* rows, const int64_t* cols, const void* vals, int pr, int pc,
                           int only_rank, spg_block* blocks);
SPG_API void spg_block_free(spg_block* b);

/* gather (dist_matrix.hpp gather): every rank's CSC block of C
 * (block-local indices, rows offset row_off, columns offset col_off) to world
 * rank `root`, assembled there ON THE GPU into the full nrows x ncols CSC
 * matrix (blocks over NCCL send/recv; columns merged in block-row order).
 * Collective over all ranks; non-root ranks get an empty `out`. */
SPG_API int spg_gather(spg_comm* comm, spg_ctx* ctx, int sr, const spg_dcsr* block_csc, int64_t row_off,
                       int64_t col_off, int64_t nrows, int64_t ncols, int root, spg_dcsr* out_csc);

#ifdef __cplusplus
}
#endif
#endif /* SPGEMM_B200_H */
