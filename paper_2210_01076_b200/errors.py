"""Exception hierarchy mirroring the reference (types.hpp:21-64).

QT_ERR_* status codes of include/qtask_c.h map one-to-one onto these.
"""


class Error(RuntimeError):
    """qtask::Error -- base of all circuit / engine errors."""


class NetConflictError(Error):
    pass


class UnknownNetError(Error):
    pass


class UnknownGateError(Error):
    pass


class BadQubitError(Error):
    pass


class InvalidPositionError(Error):
    pass


class StaleStateError(Error):
    pass


class NumericError(Error):
    pass


class SuperpositionGateError(Error):
    pass


class CudaError(Error):
    """Device-side failure (no reference counterpart)."""


class OutOfMemoryError(CudaError):
    pass


class NcclError(CudaError):
    pass


class NoDeviceError(CudaError):
    pass


_BY_CODE = {
    -1: Error, -2: NetConflictError, -3: UnknownNetError, -4: UnknownGateError,
    -5: BadQubitError, -6: InvalidPositionError, -7: StaleStateError, -8: NumericError,
    -9: SuperpositionGateError, -20: CudaError, -21: OutOfMemoryError, -22: NcclError,
    -23: NoDeviceError,
}


def from_code(code: int, msg: str) -> Error:
    return _BY_CODE.get(code, Error)(f"{msg} (status {code})")
