"""Exception types of the drop-in API (mirror dynlp/errors.py:1-9).

The C-ABI returns status codes (include/dynlp_b200.h); the host layer maps
them onto these classes: 3 -> ValidationError, 4 -> FileFormatError,
5 -> CudaError, 6 -> InternalError.
"""


class ValidationError(ValueError):
    """Input violates a documented precondition or invariant."""


class FileFormatError(ValueError):
    """An input file does not parse as its documented format."""


class CudaError(RuntimeError):
    """The device path failed (launch, allocation or driver error)."""


class InternalError(RuntimeError):
    """An engine invariant was violated."""
