// Device layout helpers that only depend on the value WIDTH, not on the
// semiring: index narrowing/widening at the host boundary, panel slicing
// (csr_row_slice / csr_col_slice, summa.hpp:57-98) into the contiguous
// broadcast wire format, and DCSC decompression (formats.hpp:220-250).
//
// Wire format of one panel (K6): a single contiguous device buffer
//   int64 rowptr[rows + 1] | pad16 | int32 colids[nnz] | pad16 | values[nnz]
// so a received message is used in place as a CSR (no deserialisation).
#pragma once
#include "common.cuh"

namespace spg {

inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

inline size_t panel_bytes(int64_t rows, int64_t nnz, int vs) {
  return align16(sizeof(int64_t) * (rows + 1)) + align16(sizeof(int32_t) * nnz) + (size_t)vs * nnz;
}

inline spg_dcsr panel_view(void* buf, int64_t rows, int64_t cols, int64_t nnz) {
  spg_dcsr v;
  v.nrows = rows;
  v.ncols = cols;
  v.nnz = nnz;
  char* p = static_cast<char*>(buf);
  v.ptr = reinterpret_cast<int64_t*>(p);
  p += align16(sizeof(int64_t) * (rows + 1));
  v.idx = reinterpret_cast<int32_t*>(p);
  p += align16(sizeof(int32_t) * nnz);
  v.vals = p;
  return v;
}

// Value-width carrier types.
template <int VS>
struct VBytes;
template <>
struct VBytes<1> { using T = uint8_t; };
template <>
struct VBytes<2> { using T = uint16_t; };
template <>
struct VBytes<4> { using T = uint32_t; };
template <>
struct VBytes<8> { using T = unsigned long long; };
template <>
struct VBytes<16> { using T = uint4; };

template <class F>
void with_vs(int vs, F&& f) {
  switch (vs) {
    case 1: f(VBytes<1>{}); break;
    case 2: f(VBytes<2>{}); break;
    case 4: f(VBytes<4>{}); break;
    case 8: f(VBytes<8>{}); break;
    case 16: f(VBytes<16>{}); break;
    default: fail(SPG_ERR_ARG, "unsupported value size " + std::to_string(vs));
  }
}

struct SrOps;
// distribute + coo_to_csc on the device (distribute.cu); host arrays of the
// blocks come from `halloc`.
void distribute_coo(spg_ctx* c, const SrOps* ops, int64_t nrows, int64_t ncols, int64_t nnz, const int64_t* rows,
                    const int64_t* cols, const void* vals, int pr, int pc, int only_rank, spg_block* blocks,
                    void* (*halloc)(size_t));

void narrow_indices(spg_ctx* c, const int64_t* in, int32_t* out, int64_t n, int64_t bound);
void widen_indices(spg_ctx* c, const int32_t* in, int64_t* out, int64_t n);
// out.rowptr[r] = m.rowptr[b + r] - m.rowptr[b]; idx/vals copied.
void slice_rows_into(spg_ctx* c, const spg_dcsr& m, int64_t b, int64_t e, int vs, const spg_dcsr& out);
// per-row count of columns in [b, e) into cnt[0 .. nrows), cnt[nrows] = 0
void slice_cols_count(spg_ctx* c, const spg_dcsr& m, int64_t b, int64_t e, int64_t* cnt);
// after rowptr = exclusive_scan(cnt): copy kept entries with columns rebased
void slice_cols_fill(spg_ctx* c, const spg_dcsr& m, int64_t b, int64_t e, int vs, const spg_dcsr& out);
// DCSC (jc, cp) -> CSC colptr on device; jc/cp already on device
void dcsc_colptr(spg_ctx* c, int64_t ncols, int64_t njc, const int64_t* jc, const int64_t* cp,
                 int64_t* colptr);
void exclusive_scan_i64(spg_ctx* c, const int64_t* in, int64_t* out, int64_t n);
// F_i (products of row i of L (x) R) for every row of l
void row_products(spg_ctx* c, const spg_dcsr& l, const spg_dcsr& r, int64_t* f);

// Horizontal concatenation of K CSR matrices with equal row counts: row i of
// the result is row i of part 0, then part 1, ... with part p's columns shifted
// by col_shift[p].  Vertical concatenation (stacking rows) of K CSRs.  Both
// allocate `out` from the context pool.
void concat_cols(spg_ctx* c, int K, const spg_dcsr* parts, const int64_t* col_shift, int vs, spg_dcsr* out);
void concat_rows(spg_ctx* c, int K, const spg_dcsr* parts, int64_t ncols, int vs, spg_dcsr* out);
void inclusive_scan_i64(spg_ctx* c, const int64_t* in, int64_t* out, int64_t n);

}  // namespace spg
