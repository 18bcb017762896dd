"""Exception classes mirroring the reference (proj/include/spsumma/common.hpp:12-73).

The C-ABI returns an SPG_ERR_* status; `from_status` maps it onto the class the
reference would have thrown for the same condition.
"""


class Error(RuntimeError):
    """spsumma::Error (common.hpp:14-17)."""


class MalformedInputError(Error):
    pass


class UnsupportedFormatError(Error):
    pass


class ShapeError(Error):
    pass


class GridError(Error):
    pass


class UnsupportedSemiringError(Error):
    pass


class ProtocolError(Error):
    pass


class DeadlockError(Error):
    pass


class AbortedError(Error):
    pass


class InvalidRangeError(Error):
    pass


class InternalError(Error):
    pass


class CudaError(Error):
    """CUDA runtime failure (no reference analogue: the reference has no GPU)."""


class OutOfMemoryError(Error):
    pass


_BY_STATUS = {
    1: ShapeError, 2: GridError, 3: UnsupportedSemiringError, 4: ProtocolError,
    5: MalformedInputError, 6: InvalidRangeError, 7: InternalError, 8: AbortedError,
    9: DeadlockError, 10: CudaError, 11: OutOfMemoryError, 12: ProtocolError,
    13: ValueError, 14: UnsupportedFormatError,
}


def from_status(status: int, msg: str) -> Exception:
    cls = _BY_STATUS.get(status, Error)
    return cls(msg)
