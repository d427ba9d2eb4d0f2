"""Exception classes of the sliced-weight path, plus the C-ABI status mapping.

Every class subclasses ``ValueError`` exactly as the reference does
(/root/reference/pkg/src/sliceplan/errors.py:1-33), so ``except ValueError``
call sites keep working after the swap.  The native library
(``include/sliced.h``) reports failures as integer status codes; ``raise_for``
turns a code plus the library's thread-local message back into the matching
class.
"""

from __future__ import annotations


class SchemaViolation(ValueError):
    """A profile/model document does not follow its schema (errors.py:4-9)."""

    def __init__(self, path: str, message: str):
        self.path = path
        super().__init__(f"{path}: {message}")


class EmptySamples(ValueError):
    """Not enough profiling samples for a fit (errors.py:12-13)."""


class DegenerateSamples(ValueError):
    """Every sample has the same workload size, so no slope (errors.py:16-17)."""


class MixedOpClass(ValueError):
    """Samples of different op classes or precisions in one fit (errors.py:20-21)."""


class ShapeMismatch(ValueError):
    """Operands disagree on a shared dimension (errors.py:24-25)."""


class TokenCountOutOfRange(ValueError):
    """A diverted-token count outside [0, T] (errors.py:28-29)."""


class NonIncreasingStep(ValueError):
    """A memory-assignment step that does not raise the fraction (errors.py:32-33)."""


class NativeError(RuntimeError):
    """CUDA / allocation failure inside the native library (no reference twin:
    the reference never touches a device)."""


# Status codes returned by every sp_* entry point (include/sliced.h).
SP_OK = 0
SP_ERR_SHAPE = 1
SP_ERR_TOKENS = 2
SP_ERR_VALUE = 3
SP_ERR_CUDA = 4
SP_ERR_NOMEM = 5
SP_ERR_STATE = 6

_STATUS_CLASS = {
    SP_ERR_SHAPE: ShapeMismatch,
    SP_ERR_TOKENS: TokenCountOutOfRange,
    SP_ERR_VALUE: ValueError,
    SP_ERR_CUDA: NativeError,
    SP_ERR_NOMEM: MemoryError,
    SP_ERR_STATE: NativeError,
}


def raise_for(status: int, message: str) -> None:
    """Raise the exception class that corresponds to a native status code."""
    if status == SP_OK:
        return
    raise _STATUS_CLASS.get(status, NativeError)(message or f"native status {status}")
