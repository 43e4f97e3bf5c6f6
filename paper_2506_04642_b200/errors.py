"""Typed errors of the TaDA hot path.

Names and base classes are the reference's (pkg/src/tadakv/errors.py:4-33) so a
caller's ``except ShapeError`` / ``except ValueError`` keeps working after the
switch; the C ABI status codes map onto them in ``_lib.check``.
"""


class TadaError(Exception):
    """Root of every error raised by this package."""


class ShapeError(TadaError, ValueError):
    """Tensor dimensions disagree with the cache / config geometry."""


class ConfigError(TadaError, ValueError):
    """A width, geometry or policy parameter is invalid."""


class DataError(TadaError, ValueError):
    """Values the quantizer cannot represent (NaN / inf)."""


class FormatError(TadaError, ValueError):
    """A packed record or TADAKV1 blob is malformed or truncated."""


class StateError(TadaError, RuntimeError):
    """The call does not fit the current cache state (e.g. attending an empty cache)."""


class CapacityError(TadaError, RuntimeError):
    """A fixed capacity (pages, residual slots) would overflow."""


class BudgetInfeasibleError(TadaError, RuntimeError):
    """Kept for API compatibility with the reference's precision search."""
