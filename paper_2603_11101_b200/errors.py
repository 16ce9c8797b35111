"""Python mirror of the reference's exception taxonomy (proj/include/vlasim/util/errors.hpp:8-39).

C-ABI status codes (include/vlasim_cuda.h) map as: 2 → ConfigError, 3 → SimError, 4 → InternalError.
"""


class ConfigError(ValueError):
    """Bad user input (errors.hpp:8-12): oversize samples, bad shapes, bad capacity. CLI exit 2."""


class SimError(RuntimeError):
    """Runtime failure while executing (errors.hpp:14-18): CUDA/NCCL errors. CLI exit 3."""


class InternalError(AssertionError):
    """Violated internal invariant (errors.hpp:35-39). Always a bug."""


def raise_for_status(code: int, msg: str) -> None:
    if code == 0:
        return
    if code == 2:
        raise ConfigError(msg)
    if code == 4:
        raise InternalError(msg)
    raise SimError(msg)
