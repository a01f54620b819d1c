"""Exception types of the criterion path, named as in the reference
(pkg/src/asrkit/errors.py:4-54) so callers' ``except`` clauses keep working.

The C-ABI status codes (include/w2l_criterion.h) map onto them 1:1 through
``raise_for_status``.
"""


class AsrkitError(Exception):
    """Base class for all toolkit errors (errors.py:4)."""


class ContractError(AsrkitError):
    """An API precondition was violated by the caller (errors.py:12)."""


class NumericError(AsrkitError):
    """Non-finite values where finite ones are required (errors.py:16)."""


class TokenError(AsrkitError):
    """Unknown token symbol or id (errors.py:41)."""


class TargetError(AsrkitError):
    """A training target violates the active criterion's constraints (errors.py:49)."""


class InfeasibleTargetError(TargetError):
    """No framewise alignment of the target exists for the given length (errors.py:53)."""


class EmissionsFormatError(AsrkitError):
    """Corrupt or incompatible emissions binary file (errors.py:78)."""


class DeviceError(AsrkitError):
    """CUDA launch/runtime failure or collective failure in the native layer."""


# C-ABI status code -> exception class
STATUS_CLASSES = {
    1: ContractError,
    2: NumericError,
    3: TargetError,
    4: InfeasibleTargetError,
    5: DeviceError,
    6: DeviceError,
    7: NumericError,
}


def raise_for_status(code: int, message: str) -> None:
    if code == 0:
        return
    raise STATUS_CLASSES.get(code, DeviceError)(message)
