"""Exception classes of the drop-in API.

When the reference package (`symfuse`) is importable its classes are re-used,
so `except SymfuseError` clauses inside the unchanged reference code (e.g.
random_equiv_test, interp.py:268-281) catch errors raised by this backend.
Otherwise an identically named hierarchy is defined (errors.py:1-38).
"""
from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from symfuse.errors import (  # type: ignore
        ConstraintError,
        DeserializeError,
        DivisibilityError,
        EmptyParamSpaceError,
        NonIntegerError,
        ResourceLimitError,
        ShapeError,
        SymfuseError,
        UnsupportedOpError,
        WriteConflictError,
    )
except ImportError:  # the GPU box carries no reference install
    class SymfuseError(Exception):
        """Base class (symfuse errors.py:1)."""

    class ShapeError(SymfuseError):
        pass

    class DivisibilityError(SymfuseError):
        pass

    class NonIntegerError(DivisibilityError):
        pass

    class ConstraintError(SymfuseError):
        pass

    class DeserializeError(SymfuseError):
        pass

    class UnsupportedOpError(SymfuseError):
        pass

    class EmptyParamSpaceError(SymfuseError):
        pass

    class WriteConflictError(SymfuseError):
        pass

    class ResourceLimitError(SymfuseError):
        pass


class KernelTimeout(ResourceLimitError):
    """The generated kernel's watchdog fired (a wait on an asynchronous completion
    exceeded 2 s); a SymfuseError, so random_equiv_test reports "run: ..."."""


class BackendError(RuntimeError):
    """CUDA / NVRTC failure inside libsgm (status >= 100)."""


class BackendUnavailable(BackendError):
    """libsgm.so or a B200 is missing.  There is no CPU fallback by design."""


def from_status(status: int, message: str) -> Exception:
    """Map an sgm_status (include/sgm.h) to the reference's exception class."""
    table = {
        1: ShapeError,
        2: DivisibilityError,
        3: WriteConflictError,
        4: UnsupportedOpError,
        5: ConstraintError,
        6: ValueError,  # numpy raises ValueError for contraction / broadcast mismatches
    }
    cls = table.get(status, BackendError)
    return cls(message)
