"""Exception types mirroring the reference's error conventions.

Reference: `numerics.py:20-29` (DimensionError, DomainError, NonFiniteError).
The C-ABI status codes (include/accel.h) map onto these one-to-one.
"""

from __future__ import annotations


class DimensionError(ValueError):
    """Shape mismatch; the message names the offending tensor (numerics.py:20-21)."""


class DomainError(ValueError):
    """Input outside a function's domain (numerics.py:24-25)."""


class NonFiniteError(ValueError):
    """NaN or infinity where a finite value is required (numerics.py:28-29)."""


class PayloadError(ValueError):
    """Malformed inference batch: empty or mixed kinds (inference.py:38-39)."""


class AccelError(RuntimeError):
    """CUDA-side failure (status 4) or a missing native library."""


STATUS_OK = 0
STATUS_DOMAIN = 1
STATUS_DIMENSION = 2
STATUS_NONFINITE = 3
STATUS_CUDA = 4

_STATUS_EXC = {
    STATUS_DOMAIN: DomainError,
    STATUS_DIMENSION: DimensionError,
    STATUS_NONFINITE: NonFiniteError,
    STATUS_CUDA: AccelError,
}


def raise_for_status(status: int, message: str) -> None:
    if status == STATUS_OK:
        return
    raise _STATUS_EXC.get(status, AccelError)(message or f"accel status {status}")
