"""Exception types of the criterion path, named as in the reference
(pkg/src/asrkit/errors.py:4-54) so callers' ``except`` clauses keep working.

The C-ABI status codes (include/w2l_criterion.h) map onto them 1:1 through
``raise_for_status``.
"""

import importlib
import os


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


# Drop-in mode: with W2L_REFERENCE_ERRORS naming the reference's errors
# module (e.g. "asrkit.errors"), the shim raises the reference's own classes,
# so existing ``except``/``pytest.raises`` clauses written against the
# reference catch them (tools/ref_suite.py runs the reference tests so).
_REF = os.environ.get("W2L_REFERENCE_ERRORS")
if _REF:
    _ref = importlib.import_module(_REF)
    AsrkitError = _ref.AsrkitError
    ContractError = _ref.ContractError
    NumericError = _ref.NumericError
    TokenError = _ref.TokenError
    TargetError = _ref.TargetError
    InfeasibleTargetError = _ref.InfeasibleTargetError
    EmissionsFormatError = _ref.EmissionsFormatError

    class DeviceError(AsrkitError):  # noqa: F811  (not in the reference)
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
