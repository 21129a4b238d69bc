"""Exception types of the drop-in surface (reference: connlab/errors.py:4-13).

The C ABI reports GC_ERR_CONFIG / GC_ERR_MALFORMED status codes; the ctypes
layer turns them into these, so callers catch exactly what they caught with
the CPU reference.
"""


class ConfigError(ValueError):
    """Invalid algorithm specification or parameter combination."""


class MalformedInputError(ValueError):
    """Graph or edge-list input that violates its format contract."""


class VerificationError(AssertionError):
    """A result failed an oracle / forest / prefix check."""


class NativeError(RuntimeError):
    """libgconn reported a CUDA or resource failure (no CPU fallback exists)."""
