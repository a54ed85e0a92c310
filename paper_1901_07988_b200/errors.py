"""Error taxonomy of the package and the C-ABI status mapping.

The class names and bases are those of the reference package
(/root/reference/pkg/src/qtape/errors.py:4-29) so callers that catch
``ShapeError`` / ``ConfigError`` / ... keep working; device failures reported
by the CUDA library surface as ``StateError`` carrying the CUDA message.
"""


class QtapeError(Exception):
    """Root of every error raised by this package."""


class ShapeError(QtapeError, ValueError):
    """Extents violate an operator's shape contract."""


class ConfigError(QtapeError, ValueError):
    """Unsupported configuration (bit width, width > 2, schedule, dtype)."""


class CodecError(QtapeError, ValueError):
    """Packing called with out-of-range codes or a wrong byte count."""


class StateError(QtapeError, RuntimeError):
    """Tape / parameter / device state inconsistent with the request."""


class DataError(QtapeError, ValueError):
    """Dataset content violates an invariant (e.g. a label out of range)."""


class FormatError(DataError):
    """A data file is not in the expected binary layout."""


# Status codes of include/qtape_b200.h
QT_OK = 0
QT_EINVAL = -1
QT_EUNSUPPORTED = -2


def raise_for_status(status: int, fn: str, message: str) -> None:
    """Translate a nonzero qt_* return code into an exception (never a
    silent fallback: contrast _native.py:67-68 of the reference)."""
    if status == QT_OK:
        return
    if status == QT_EINVAL:
        raise ShapeError(f"{fn}: {message}")
    if status == QT_EUNSUPPORTED:
        raise ConfigError(f"{fn}: {message}")
    raise StateError(f"{fn}: CUDA error {status}: {message}")
