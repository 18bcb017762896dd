"""B200-native distributed semiring SpGEMM (drop-in for the spsumma reference API).

The compute path is hand-written sm_100a CUDA behind the C-ABI in
include/spgemm_b200.h (libspgemm_b200.so in this package directory).
"""
from . import errors
from ._lib import lib
from .device import Context, DeviceCsr, default_context
from .formats import (CooMatrix, CscMatrix, CsrMatrix, DcscMatrix, coo_to_csc, coo_to_csr, csc_to_coo,
                      csc_to_csr, csc_to_dcsc, csr_to_coo, csr_to_csc, dcsc_decompress,
                      reinterpret_transpose, validate)
from .generators import generate_er, generate_rmat, generate_stencil27
from .matrix_market import read_matrix_market
from .local_spgemm import esc_multiply, local_multiply, matrix_checksum, merge_partials
from .semiring import SemiringId, dtype_of, register_semiring, semiring_by_name

__all__ = [
    "errors", "lib", "Context", "DeviceCsr", "default_context", "CooMatrix", "CscMatrix", "CsrMatrix",
    "DcscMatrix", "coo_to_csc", "coo_to_csr", "csc_to_coo", "csc_to_csr", "csc_to_dcsc", "csr_to_coo",
    "csr_to_csc", "dcsc_decompress", "reinterpret_transpose", "validate", "generate_er", "generate_rmat",
    "generate_stencil27", "esc_multiply", "local_multiply", "matrix_checksum", "merge_partials",
    "SemiringId", "dtype_of", "register_semiring", "semiring_by_name", "read_matrix_market",
]
