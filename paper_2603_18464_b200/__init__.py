"""B200-native AcceRL trainer hot path (drop-in for asyncrl.trainer).

Host side mirrors the reference Python API; the math runs in libaccel.so
(hand-written sm_100a CUDA behind the C ABI in include/accel.h).
"""

from .errors import AccelError, DimensionError, DomainError, NonFiniteError

__version__ = "0.1.0"

__all__ = ["AccelError", "DimensionError", "DomainError", "NonFiniteError", "__version__"]
