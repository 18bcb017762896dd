"""Semiring registry (mirror of proj/include/spsumma/semiring.hpp:122-149).

The device functors live in csrc/semiring.cuh; this module only names them
and gives each value type its numpy dtype (the ValueCodec byte layout,
serialize.hpp:29-76: little-endian fixed width, bool = 1 byte).
"""
from __future__ import annotations

import enum

import numpy as np

from . import errors


class SemiringId(enum.IntEnum):
    arithmetic = 0
    minplus = 1
    boolean = 2
    minselect = 3
    tropical_i32 = 4
    maxtimes = 5


MINSELECT_DTYPE = np.dtype([("weight", "<f8"), ("payload", "<i8")])
MAXTIMES_DTYPE = np.dtype([("w", "<f8"), ("tag", "<u8")])

DTYPES = {
    SemiringId.arithmetic: np.dtype("<f8"),
    SemiringId.minplus: np.dtype("<f8"),
    SemiringId.boolean: np.dtype("u1"),
    SemiringId.minselect: MINSELECT_DTYPE,
    SemiringId.tropical_i32: np.dtype("<i4"),
    SemiringId.maxtimes: MAXTIMES_DTYPE,
}

COMMUTATIVE = {s: s != SemiringId.minselect for s in SemiringId}

# user-defined semirings registered at run time: id -> (name, dtype, library handle)
_USER = {}


def register_semiring(library_path: str, symbol: str, dtype) -> int:
    """Load a user semiring library — a .cu with SPG_INSTANTIATE(MySemiring,
    symbol) compiled against this repo's headers (tests/custom_sr/ is an
    example) — and register its ops table (spg_register_semiring).  Returns
    the semiring id every entry point then accepts; `dtype` is the numpy
    view of its value_type (the ValueCodec byte layout)."""
    import ctypes as C

    from ._lib import check, lib
    handle = C.CDLL(library_path)
    fn = getattr(handle, symbol)
    fn.restype = C.c_void_p
    sid = C.c_int()
    check(lib.spg_register_semiring(C.c_void_p(fn()), C.byref(sid)))
    dt = np.dtype(dtype)
    vs = int(lib.spg_value_size(sid.value))
    if dt.itemsize != vs:
        raise errors.ShapeError(f"dtype {dt} is {dt.itemsize} bytes, the semiring's value_type is {vs}")
    _USER[sid.value] = (lib.spg_semiring_name(sid.value).decode(), dt, handle)
    return sid.value


def semiring_by_name(name: str):
    """semiring_by_name (semiring.hpp:125-133); MalformedInputError if unknown."""
    try:
        return SemiringId[name]
    except KeyError:
        for sid, (n, _, _) in _USER.items():
            if n == name:
                return sid
        raise errors.MalformedInputError(
            f"unknown semiring '{name}' (expected arithmetic, minplus, boolean, minselect, "
            "tropical_i32, or maxtimes)") from None


def as_id(sr):
    if isinstance(sr, str):
        return semiring_by_name(sr)
    if int(sr) in _USER:
        return int(sr)
    return SemiringId(int(sr))


def dtype_of(sr) -> np.dtype:
    sid = as_id(sr)
    if sid in _USER:
        return _USER[sid][1]
    return DTYPES[sid]


def zero(sr):
    """SR::zero() as a numpy scalar of the semiring's dtype."""
    sr = as_id(sr)
    dt = DTYPES[sr]
    if sr == SemiringId.arithmetic:
        return dt.type(0.0)
    if sr == SemiringId.minplus:
        return dt.type(np.inf)
    if sr == SemiringId.boolean:
        return dt.type(0)
    if sr == SemiringId.tropical_i32:
        return dt.type(np.iinfo(np.int32).max)
    if sr == SemiringId.minselect:
        return np.array([(np.inf, np.iinfo(np.int64).max)], dtype=dt)[0]
    return np.array([(0.0, 0)], dtype=dt)[0]


def from_real(sr, x):
    """SR::from_real applied elementwise to a float array."""
    sr = as_id(sr)
    x = np.asarray(x, dtype=np.float64)
    if sr in (SemiringId.arithmetic, SemiringId.minplus):
        return x.copy()
    if sr == SemiringId.boolean:
        return (x != 0).astype(np.uint8)
    if sr == SemiringId.tropical_i32:
        y = x * 1024.0
        out = np.where(y >= 2147483646.5, 2147483647,
                       np.where(y < -2147483648.0, -2147483648,
                                np.sign(y) * np.floor(np.abs(y) + 0.5)))
        return out.astype(np.int32)
    out = np.zeros(x.shape, dtype=DTYPES[sr])
    if sr == SemiringId.minselect:
        out["weight"] = x
        out["payload"] = 0
    else:
        out["w"] = x
        out["tag"] = 0
    return out
