"""Exception taxonomy of the voxsplat API, plus the C-ABI status mapping.

The names are the public contract callers catch (reference:
``voxsplat/errors.py:8-57``); every native entry point in ``include/vsx_b200.h``
returns an integer status that :func:`raise_for_status` turns into one of them.
"""

from __future__ import annotations


class VoxsplatError(Exception):
    """Root of every error raised by this package."""


class InvalidInput(VoxsplatError):
    """Arguments violate a documented precondition (shape, range, ordering)."""


class IoError(VoxsplatError):
    """A file could not be read or written."""


class NumericalError(VoxsplatError):
    """Non-finite output, or a 2D covariance that is not positive definite."""


class ResourceError(VoxsplatError):
    """A device allocation or capacity budget was exceeded."""


class StateError(VoxsplatError):
    """Call sequence error, e.g. a backward without a recorded forward."""


class ProtocolError(VoxsplatError):
    """Ranks or replicas disagree (collective participants, replica bits)."""


class TransferError(VoxsplatError):
    """A rank that owns gaussians needed by a view is unreachable."""


class ContractViolation(VoxsplatError):
    """An ordering/shape contract between pipeline stages was broken."""


class InsufficientData(VoxsplatError):
    """Too few samples for a fit (reference errors.py:44)."""


class DegenerateFit(VoxsplatError):
    """A fit has no unique / admissible solution (reference errors.py:48)."""


# Status codes shared with include/vsx_b200.h (VSX_OK ... VSX_ERR_CUDA).
VSX_OK = 0
VSX_ERR_INVALID = -1
VSX_ERR_NUMERICAL = -2
VSX_ERR_CONTRACT = -3
VSX_ERR_CUDA = -4
VSX_ERR_CAPACITY = -5

_STATUS_TO_ERROR = {
    VSX_ERR_INVALID: InvalidInput,
    VSX_ERR_NUMERICAL: NumericalError,
    VSX_ERR_CONTRACT: ContractViolation,
    VSX_ERR_CUDA: RuntimeError,
    VSX_ERR_CAPACITY: ResourceError,
}


def raise_for_status(code: int, what: str, detail: str = "") -> None:
    """Translate a native status code into the matching exception."""
    if code == VSX_OK:
        return
    exc = _STATUS_TO_ERROR.get(code, RuntimeError)
    msg = f"{what} failed (status {code})"
    if detail:
        msg += f": {detail}"
    raise exc(msg)
