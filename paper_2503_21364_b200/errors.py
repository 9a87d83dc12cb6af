"""Error types mirroring the reference's (all ValueError subclasses).

Reference: pkg/src/landmark/common.py:14-31.  The Python wrappers pre-validate
inputs and raise these so callers that catch the reference's exceptions keep
working; C-ABI failures surface as ``LmgsError`` (a RuntimeError) carrying the
library's error string.
"""


class InvalidConfigError(ValueError):
    pass


class InvalidInputError(ValueError):
    pass


class ShapeError(ValueError):
    pass


class OutOfBoundsError(ValueError):
    pass


class FormatError(ValueError):
    pass


class LmgsError(RuntimeError):
    """A failure reported by the native library (CUDA error, bad argument)."""
