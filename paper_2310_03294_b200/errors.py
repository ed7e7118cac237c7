"""Exception taxonomy of /root/reference/proj/include/distattn/errors.hpp:12-48,
mapped from the C ABI status codes (include/distattn_b200.h)."""
from __future__ import annotations


class Error(RuntimeError):
    """distattn::Error"""


class ShapeError(Error):
    """Operand dimensions do not match the operation's contract."""


class ConfigError(Error):
    """Invalid configuration value (zero workers, non-divisible split, ...)."""


class ScheduleError(Error):
    """A schedule failed validation or does not fit the shards."""


class StateError(Error):
    """An operation was invoked before its required state exists."""


class DegenerateRowError(Error):
    """A softmax row absorbed no keys."""


class CudaError(Error):
    """CUDA runtime or launch failure inside the library."""


class NcclError(Error):
    """NCCL failure in the distributed runtime."""


class UnsupportedError(Error):
    """Shape outside what the sm_100a kernels implement (d != 128, ...)."""


STATUS = {1: ShapeError, 2: ConfigError, 3: ScheduleError, 4: StateError, 5: DegenerateRowError,
          6: CudaError, 7: NcclError, 8: UnsupportedError}


def check(status: int) -> None:
    if status == 0:
        return
    from . import _lib
    msg = _lib.lib().da_last_error()
    msg = msg.decode() if msg else ""
    raise STATUS.get(status, Error)(msg or f"distattn status {status}")
