"""Exception taxonomy of the reference (common.hpp:22-36), raised from ABI status codes."""


class MPMError(RuntimeError):
    pass


class ValidationError(MPMError):
    """common.hpp:24-26 (CLI exit code 2)."""


class NumericalError(MPMError):
    """common.hpp:28-30 (CLI exit code 3)."""


class OutOfDomainError(NumericalError):
    """common.hpp:32-36: carries the offending particle index."""

    def __init__(self, particle: int, what: str):
        super().__init__(what)
        self.particle = particle


class DeviceError(MPMError):
    """CUDA / NCCL failure (ABI status 6); there is no CPU fallback."""


def raise_for(code: int, particle: int, msg: str):
    if code == 0:
        return
    if code == 2:
        raise ValidationError(msg)
    if code == 4:
        raise OutOfDomainError(particle, msg)
    if code in (3, 5):
        raise NumericalError(msg)
    if code == 6:
        raise DeviceError(msg)
    raise MPMError(f"status {code}: {msg}")
