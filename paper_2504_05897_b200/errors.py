"""Exception types of the reference API, shared by every module.

Same names and bases as the reference: EvictionError(RuntimeError)
(caching.py:26-27), PlanInvariantError(ValueError) (scheduling.py:76-77),
CalibrationError(ValueError) (costs.py:98-99), TraceFormatError(ValueError)
(tracegen.py:298-299).
"""


class EvictionError(RuntimeError):
    """Cache full and every resident expert is pinned."""


class PlanInvariantError(ValueError):
    """A produced plan violated a schedule invariant."""


class CalibrationError(ValueError):
    """Raised when the sample set cannot determine some profile parameter."""


class TraceFormatError(ValueError):
    """Malformed trace file; message carries the line number and field."""
