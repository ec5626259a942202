"""Exception hierarchy of the skewstream API (reference errors.py:4-29).

The C-ABI reports failures as integer status codes (include/ss_b200.h,
``SS_E_*``); ``raise_for_status`` maps them onto these classes so callers
written against the reference catch the same types.
"""


class SkewStreamError(Exception):
    """Root of every error raised by this package."""


class InvalidSpecError(SkewStreamError, ValueError):
    """Malformed dataset description."""


class InvalidConfigError(SkewStreamError, ValueError):
    """Malformed run / balancer / engine configuration."""


class DataError(SkewStreamError, ValueError):
    """Tuple data violates a precondition (unknown group or key, bad file)."""


class ConsistencyError(SkewStreamError, RuntimeError):
    """Bookkeeping disagrees with itself (stale stats, split grouped run)."""


class StaleMoveError(SkewStreamError, RuntimeError):
    """A move names a group its source partition no longer owns."""


class ExecutionError(SkewStreamError, RuntimeError):
    """The device (CUDA / NCCL) failed while executing a batch."""


# status codes of include/ss_b200.h
SS_OK = 0
SS_E_DATA = 1
SS_E_CONFIG = 2
SS_E_SPEC = 3
SS_E_CONSISTENCY = 4
SS_E_STALE_MOVE = 5
SS_E_EXEC = 6

_BY_CODE = {
    SS_E_DATA: DataError,
    SS_E_CONFIG: InvalidConfigError,
    SS_E_SPEC: InvalidSpecError,
    SS_E_CONSISTENCY: ConsistencyError,
    SS_E_STALE_MOVE: StaleMoveError,
    SS_E_EXEC: ExecutionError,
}


def raise_for_status(code: int, message: str) -> None:
    if code == SS_OK:
        return
    raise _BY_CODE.get(code, ExecutionError)(message)
