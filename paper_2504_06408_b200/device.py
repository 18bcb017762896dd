"""Per-GPU context and device-resident matrices (C-ABI handles).

A `Context` is the spg_ctx of one GPU: its stream and stream-ordered memory
pool.  A `DeviceCsr` owns one spg_dcsr (int64 offsets, int32 indices).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import DCsr, HCsr, check, lib
from .formats import CscMatrix, CsrMatrix
from .semiring import as_id, dtype_of


class Context:
    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        check(lib.spg_ctx_create(device, C.byref(h)))
        self.handle = h

    @property
    def stream(self) -> int:
        return lib.spg_ctx_stream(self.handle) or 0

    def sync(self):
        check(lib.spg_ctx_sync(self.handle), self.handle)

    def kernel_launches(self) -> int:
        return int(lib.spg_ctx_kernel_launches(self.handle))

    def set_scratch_budget(self, nbytes: int):
        check(lib.spg_ctx_set_scratch_budget(self.handle, int(nbytes)), self.handle)

    PIPE_AUTO, PIPE_BINS, PIPE_SORTED = 0, 1, 2

    def set_pipeline(self, mode: int):
        """PIPE_AUTO: bitmap-rank kernels for long rows when the output width
        fits; PIPE_BINS: the per-bin accumulators with scratch + compaction;
        PIPE_SORTED: PIPE_BINS with every dense-panel row on the sort fallback
        (bin 11, otherwise only for outputs too wide for dense panels)."""
        check(lib.spg_ctx_set_pipeline(self.handle, int(mode)), self.handle)

    def close(self):
        if self.handle:
            lib.spg_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default = {}


def default_context(device: int = 0) -> Context:
    if device not in _default:
        _default[device] = Context(device)
    return _default[device]


def _hcsr(ptr, idx, vals, nrows, ncols):
    ptr = np.ascontiguousarray(ptr, dtype=np.int64)
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    vals = np.ascontiguousarray(vals)
    h = HCsr(nrows, ncols, idx.shape[0], ptr.ctypes.data_as(C.POINTER(C.c_int64)),
             idx.ctypes.data_as(C.POINTER(C.c_int64)), vals.ctypes.data_as(C.c_void_p))
    return h, (ptr, idx, vals)  # keep the arrays alive with the struct


def hcsr_of(m):
    if isinstance(m, CsrMatrix):
        return _hcsr(m.rowptr, m.colids, m.values, m.nrows, m.ncols)
    return _hcsr(m.colptr, m.rowids, m.values, m.nrows, m.ncols)


def copy_out(ptr, n: int, dt) -> np.ndarray:
    """Copy n values of dtype dt from a raw host pointer (any size; ctypes'
    string_at truncates sizes to a C int)."""
    dt = np.dtype(dt)
    if n == 0 or not ptr:
        return np.zeros(0, dtype=dt)
    raw = np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint8)), shape=(n * dt.itemsize,))
    return raw.copy().view(dt)


class _HostBlock:
    """Owns one library-allocated host array (pinned, recycled on release)."""

    __slots__ = ("ptr", "__array_interface__")

    def __init__(self, ptr, nbytes):
        self.ptr = ptr
        self.__array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}

    def __del__(self):
        if self.ptr:
            lib.spg_free(C.c_void_p(self.ptr))
            self.ptr = None


def view_owned(ptr, n: int, dt) -> np.ndarray:
    """Zero-copy numpy view of n values at a library-allocated pointer; the
    memory returns to the library when the array is garbage collected."""
    dt = np.dtype(dt)
    addr = C.cast(ptr, C.c_void_p).value
    if not addr:
        return np.zeros(n, dtype=dt)
    raw = np.asarray(_HostBlock(addr, max(n, 1) * dt.itemsize))
    return raw[: n * dt.itemsize].view(dt)


def pinned_copy(a: np.ndarray) -> np.ndarray:
    """Copy of `a` in page-locked host memory from the library's pinned
    cache (uploads from it run at full PCIe speed; no cudaHostRegister, whose
    page locking the host may cap)."""
    a = np.ascontiguousarray(a)
    p = lib.spg_host_alloc(max(a.nbytes, 1))
    if not p:
        raise MemoryError(f"spg_host_alloc({a.nbytes}) failed")
    out = view_owned(C.c_void_p(p), a.size, a.dtype).reshape(a.shape)
    np.copyto(out, a)
    return out


def take_hcsr(sr, h: HCsr, is_csc: bool):
    """Wrap a library-allocated spg_hcsr as numpy arrays (zero copy)."""
    nseg = h.ncols if is_csc else h.nrows
    nnz = int(h.nnz)
    dt = dtype_of(sr)
    ptr = view_owned(h.ptr, nseg + 1, np.int64)
    idx = view_owned(h.idx, nnz, np.int64)
    vals = view_owned(h.vals, nnz, dt)
    if is_csc:
        return CscMatrix(int(as_id(sr)), int(h.nrows), int(h.ncols), ptr, idx, vals)
    return CsrMatrix(int(as_id(sr)), int(h.nrows), int(h.ncols), ptr, idx, vals)


class DeviceCsr:
    """A device CSR (or CSC when is_csc) owned by a Context."""

    def __init__(self, ctx: Context, sr, d: DCsr, is_csc: bool = False):
        self.ctx = ctx
        self.sr = as_id(sr)
        self.d = d
        self.is_csc = is_csc

    @classmethod
    def upload(cls, ctx: Context, m) -> "DeviceCsr":
        is_csc = isinstance(m, CscMatrix)
        h, keep = hcsr_of(m)
        d = DCsr()
        check(lib.spg_upload(ctx.handle, int(m.sr), C.byref(h), int(is_csc), C.byref(d)), ctx.handle)
        return cls(ctx, m.sr, d, is_csc)

    @property
    def nrows(self):
        return int(self.d.nrows)

    @property
    def ncols(self):
        return int(self.d.ncols)

    @property
    def nnz(self):
        return int(self.d.nnz)

    def download(self):
        h = HCsr()
        check(lib.spg_download(self.ctx.handle, int(self.sr), C.byref(self.d), int(self.is_csc), C.byref(h)),
              self.ctx.handle)
        return take_hcsr(self.sr, h, self.is_csc)

    def rowptr_host(self) -> np.ndarray:
        """The device row (CSC: column) pointers copied to the host."""
        nseg = self.ncols if self.is_csc else self.nrows
        out = np.empty(nseg + 1, dtype=np.int64)
        check(lib.spg_copy_to_host(self.ctx.handle, out.ctypes.data_as(C.c_void_p),
                                   C.c_void_p(self.d.ptr), out.nbytes), self.ctx.handle)
        return out

    def checksum(self) -> int:
        out = C.c_uint64()
        check(lib.spg_checksum(self.ctx.handle, int(self.sr), C.byref(self.d), int(self.is_csc), C.byref(out)),
              self.ctx.handle)
        return int(out.value)

    def free(self):
        if self.d is not None and self.d.ptr:
            lib.spg_dcsr_free(self.ctx.handle, C.byref(self.d))
        self.d = None

    def __del__(self):
        try:
            if self.ctx.handle is not None:
                self.free()
        except Exception:
            pass


def pin(*arrays):
    """Page-lock numpy arrays in place (cudaHostRegister) so their uploads run
    at full PCIe speed; returns a callable that unpins them.  Pinning is a
    transfer-speed hint: an array the driver refuses to lock (e.g. beyond
    the host's lockable-memory limit) stays pageable and still uploads."""
    done = []
    for a in arrays:
        if a is None or a.nbytes == 0:
            continue
        if lib.spg_host_register(C.c_void_p(a.ctypes.data), int(a.nbytes)) != 0:
            import sys
            print(f"[spg] pin: {a.nbytes} B left pageable ({lib.spg_last_error(None).decode()})", file=sys.stderr)
            continue
        done.append(a)

    def unpin():
        for a in done:
            lib.spg_host_unregister(C.c_void_p(a.ctypes.data))
    return unpin
