"""ctypes binding of the C-ABI in include/spgemm_b200.h.

The product path ALWAYS goes through libspgemm_b200.so (sm_100a kernels).
There is no CPU fallback: if the library is missing this module raises on
import, and every compute call raises when no GPU is present.
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPG_LIB_PATH") or os.path.join(_HERE, "libspgemm_b200.so")  # override: A/B builds


class HCsr(C.Structure):
    """spg_hcsr: host CSR/CSC in the reference's int64 layout."""

    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("ptr", C.POINTER(C.c_int64)), ("idx", C.POINTER(C.c_int64)),
                ("vals", C.c_void_p)]


class HDcsc(C.Structure):
    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("njc", C.c_int64), ("jc", C.POINTER(C.c_int64)), ("cp", C.POINTER(C.c_int64)),
                ("rowids", C.POINTER(C.c_int64)), ("vals", C.c_void_p)]


class Block(C.Structure):
    """spg_block: one rank's block as spg_distribute builds it."""

    _fields_ = [("row_begin", C.c_int64), ("row_end", C.c_int64), ("col_begin", C.c_int64),
                ("col_end", C.c_int64), ("is_dcsc", C.c_int), ("csc", HCsr), ("dcsc", HDcsc)]


class DCsr(C.Structure):
    """spg_dcsr: device CSR/CSC (int64 offsets, int32 indices)."""

    _fields_ = [("nrows", C.c_int64), ("ncols", C.c_int64), ("nnz", C.c_int64),
                ("ptr", C.c_void_p), ("idx", C.c_void_p), ("vals", C.c_void_p)]


class MultStats(C.Structure):
    _fields_ = [("products", C.c_int64), ("nnz_out", C.c_int64),
                ("rows_per_bin", C.c_int64 * 12), ("ms_analyse", C.c_double),
                ("ms_numeric", C.c_double), ("ms_compact", C.c_double),
                ("ms_total", C.c_double), ("kernels", C.c_int64), ("output_mode", C.c_int64),
                ("ms_symbolic", C.c_double), ("ms_fold", C.c_double), ("bitmap_bytes", C.c_int64),
                ("fold_items", C.c_int64)]

    def as_dict(self):
        return {"products": self.products, "nnz_out": self.nnz_out,
                "rows_per_bin": list(self.rows_per_bin), "ms_analyse": self.ms_analyse,
                "ms_numeric": self.ms_numeric, "ms_compact": self.ms_compact,
                "ms_total": self.ms_total, "kernels": self.kernels, "output_mode": self.output_mode,
                "ms_symbolic": self.ms_symbolic, "ms_fold": self.ms_fold, "bitmap_bytes": self.bitmap_bytes,
                "fold_items": self.fold_items}


class Stage(C.Structure):
    _fields_ = [("lo", C.c_int64), ("hi", C.c_int64), ("a_col_block", C.c_int),
                ("b_row_block", C.c_int), ("a_off", C.c_int64), ("b_off", C.c_int64)]


class SummaOpts(C.Structure):
    _fields_ = [("two_round", C.c_int), ("comm_mode", C.c_int), ("threshold", C.c_uint64),
                ("threshold_col", C.c_uint64), ("fuse_stages", C.c_int), ("output", C.c_int),
                ("batch_bytes", C.c_uint64)]


class Ledger(C.Structure):
    _fields_ = [("ms", C.c_double * 5), ("host_bcasts", C.c_uint64), ("device_bcasts", C.c_uint64),
                ("bytes_host_path", C.c_uint64), ("bytes_device_path", C.c_uint64),
                ("size_exchanges", C.c_uint64), ("local_multiply_calls", C.c_uint64),
                ("skipped_stages", C.c_uint64), ("peak_bcast_buffer_bytes", C.c_uint64),
                ("products", C.c_int64), ("ms_total", C.c_double),
                ("rooted_host_bcasts", C.c_uint64), ("rooted_device_bcasts", C.c_uint64),
                ("rooted_size_exchanges", C.c_uint64), ("checksum_part", C.c_uint64), ("nnz_out", C.c_int64),
                ("batches", C.c_int64), ("left_nnz", C.c_int64)]

    PHASES = ("prepare", "broadcast", "local_multiply", "merge", "copy")

    def as_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "ms"}
        d["ms"] = {p: self.ms[i] for i, p in enumerate(self.PHASES)}
        return d


_P = C.POINTER
_i64p = _P(C.c_int64)

# (name, restype, argtypes)
_SIGS = [
    ("spg_version", C.c_char_p, []),
    ("spg_last_error", C.c_char_p, [C.c_void_p]),
    ("spg_value_size", C.c_int, [C.c_int]),
    ("spg_semiring_by_name", C.c_int, [C.c_char_p]),
    ("spg_device_count", C.c_int, []),
    ("spg_register_semiring", C.c_int, [C.c_void_p, _P(C.c_int)]),
    ("spg_semiring_name", C.c_char_p, [C.c_int]),
    ("spg_semiring_is_commutative", C.c_int, [C.c_int]),
    ("spg_ctx_create", C.c_int, [C.c_int, _P(C.c_void_p)]),
    ("spg_ctx_destroy", None, [C.c_void_p]),
    ("spg_ctx_stream", C.c_void_p, [C.c_void_p]),
    ("spg_ctx_set_stream", C.c_int, [C.c_void_p, C.c_void_p]),
    ("spg_ctx_sync", C.c_int, [C.c_void_p]),
    ("spg_ctx_kernel_launches", C.c_uint64, [C.c_void_p]),
    ("spg_ctx_set_scratch_budget", C.c_int, [C.c_void_p, C.c_uint64]),
    ("spg_ctx_set_pipeline", C.c_int, [C.c_void_p, C.c_int]),
    ("spg_dcsr_alloc", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, _P(DCsr)]),
    ("spg_dcsr_free", C.c_int, [C.c_void_p, _P(DCsr)]),
    ("spg_copy_to_host", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64]),
    ("spg_local_multiply_rows", C.c_int, [C.c_void_p, C.c_int, _P(DCsr), _P(DCsr), C.c_int64, C.c_int64, _P(DCsr),
                                          _P(MultStats)]),
    ("spg_upload", C.c_int, [C.c_void_p, C.c_int, _P(HCsr), C.c_int, _P(DCsr)]),
    ("spg_download", C.c_int, [C.c_void_p, C.c_int, _P(DCsr), C.c_int, _P(HCsr)]),
    ("spg_hcsr_free", None, [_P(HCsr)]),
    ("spg_local_multiply", C.c_int, [C.c_void_p, C.c_int, _P(DCsr), _P(DCsr), _P(DCsr), _P(MultStats)]),
    ("spg_merge_partials", C.c_int, [C.c_void_p, C.c_int, C.c_int, _P(DCsr), _P(C.c_int), _P(C.c_int),
                                     C.c_int64, C.c_int64, _P(DCsr), _P(MultStats)]),
    ("spg_checksum", C.c_int, [C.c_void_p, C.c_int, _P(DCsr), C.c_int, _P(C.c_uint64)]),
    ("spg_checksum_part", C.c_int, [C.c_void_p, C.c_int, _P(DCsr), C.c_int, C.c_int64, C.c_int64,
                                    _P(C.c_uint64)]),
    ("spg_checksum_seed", C.c_uint64, [C.c_int64, C.c_int64]),
    ("spg_csr_slice", C.c_int, [C.c_void_p, C.c_int, _P(DCsr), C.c_int, C.c_int64, C.c_int64, _P(DCsr)]),
    ("spg_prepare_block", C.c_int, [C.c_void_p, C.c_int, _P(HCsr), _P(HDcsc), _P(DCsr)]),
    ("spg_esc_multiply", C.c_int, [C.c_void_p, C.c_int, _P(HCsr), _P(HCsr), _P(HCsr), _P(MultStats)]),
    ("spg_generate_rmat", C.c_int, [C.c_int, C.c_int, C.c_double, C.c_uint64, _i64p, _i64p,
                                    _P(_i64p), _P(_i64p), _P(C.c_void_p)]),
    ("spg_generate_er", C.c_int, [C.c_int, C.c_int64, C.c_int, C.c_uint64, C.c_int, _i64p,
                                  _P(_i64p), _P(_i64p), _P(C.c_void_p)]),
    ("spg_generate_stencil27", C.c_int, [C.c_int, C.c_int64, _i64p, _i64p, _P(_i64p), _P(_i64p),
                                         _P(C.c_void_p)]),
    ("spg_generate_er_block", C.c_int, [C.c_int, C.c_int64, C.c_int, C.c_uint64, C.c_int, C.c_int64, C.c_int64,
                                        C.c_int64, C.c_int64, _i64p, _P(_i64p), _P(_i64p), _P(C.c_void_p)]),
    ("spg_generate_stencil27_block", C.c_int, [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                               _i64p, _i64p, _P(_i64p), _P(_i64p), _P(C.c_void_p)]),
    ("spg_read_matrix_market", C.c_int, [C.c_int, C.c_char_p, _i64p, _i64p, _i64p, _P(_i64p), _P(_i64p),
                                         _P(C.c_void_p)]),
    ("spg_host_alloc", C.c_void_p, [C.c_uint64]),
    ("spg_coo_to_csr", C.c_int, [C.c_int, C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p, C.c_void_p,
                                 C.c_int, _P(HCsr)]),
    ("spg_free", None, [C.c_void_p]),
    ("spg_host_register", C.c_int, [C.c_void_p, C.c_uint64]),
    ("spg_host_unregister", C.c_int, [C.c_void_p]),
    ("spg_block_range", None, [C.c_int64, C.c_int, C.c_int, _i64p, _i64p]),
    ("spg_round_range", None, [C.c_int64, C.c_int, C.c_int, _i64p, _i64p]),
    ("spg_summa_schedule", C.c_int, [C.c_int64, C.c_int, C.c_int, _P(Stage), C.c_int]),
    ("spg_comm_create", C.c_int, [C.c_char_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                  _P(C.c_void_p)]),
    ("spg_comm_destroy", None, [C.c_void_p]),
    ("spg_comm_last_error", C.c_char_p, [C.c_void_p]),
    ("spg_comm_barrier", C.c_int, [C.c_void_p]),
    ("spg_exchange_sizes", C.c_int, [C.c_void_p, C.c_int, C.c_int, _i64p]),
    ("spg_bcast", C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_uint64, C.c_int, C.c_uint64,
                            _P(C.c_int)]),
    ("spg_comm_set_device_transport", C.c_int, [C.c_void_p, C.c_int]),
    ("spg_comm_has_device_path", C.c_int, [C.c_void_p]),
    ("spg_distribute", C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p, C.c_void_p,
                                 C.c_int, C.c_int, C.c_int, _P(Block)]),
    ("spg_block_free", None, [_P(Block)]),
    ("spg_gather", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, _P(DCsr), C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                             C.c_int, _P(DCsr)]),
    ("spg_summa25_multiply", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                       _P(HCsr), _P(HDcsc), _P(HCsr), _P(HDcsc), _P(SummaOpts),
                                       _P(DCsr), _P(Ledger)]),
]

EXPORTED = [s[0] for s in _SIGS]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -j` (or __graft_entry__.build()); "
            "there is no CPU fallback for the SpGEMM path")
    # torch first: its bundled libnccl.so.2 then satisfies this library's
    # NCCL dependency (loading the system NCCL first would leave torch's CUDA
    # library with unresolved newer NCCL symbols when it is imported later)
    try:
        import torch  # noqa: F401
    except ImportError:
        pass
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    for name, res, args in _SIGS:
        try:
            fn = getattr(lib, name)
        except AttributeError:
            MISSING.append(name)
            continue
        fn.restype = res
        fn.argtypes = args
    return lib


MISSING: list = []


lib = _load()


def check(status: int, ctx=None):
    """Raise the reference exception class matching an SPG status."""
    if status == 0:
        return
    msg = lib.spg_last_error(ctx)
    msg = msg.decode() if msg else f"status {status}"
    raise errors.from_status(status, msg)
