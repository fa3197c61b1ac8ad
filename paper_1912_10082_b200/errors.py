"""Exception classes of the reference (stk/errors.hpp:9-42) and the status-code mapping of
the C ABI (include/stk_gpu.h)."""
from __future__ import annotations


class StkError(Exception):
    """Base of all errors raised through the C ABI."""


class ArgumentError(StkError, ValueError):
    """stk::ArgumentError -- bad sizes, out-of-range arguments (stk/errors.hpp:9)."""


class DefinitenessError(StkError, RuntimeError):
    """stk::DefinitenessError -- a matrix required s.p.d. is not (stk/errors.hpp:15)."""


class SingularityError(StkError, RuntimeError):
    """stk::SingularityError -- singular row system in a structured solve (stk/errors.hpp:21)."""


class SolvabilityError(StkError, RuntimeError):
    """stk::SolvabilityError -- lambda_i + theta_j <= 0 (stk/errors.hpp:27)."""


class NumericError(StkError, RuntimeError):
    """stk::NumericError -- non-finite values during an iteration (stk/errors.hpp:33)."""


class CudaError(StkError, RuntimeError):
    """CUDA runtime failure (no reference counterpart)."""


# status codes of include/stk_gpu.h
STKG_OK, STKG_ARGUMENT, STKG_DEFINITENESS, STKG_SINGULARITY, STKG_SOLVABILITY, STKG_NUMERIC, \
    STKG_CUDA = range(7)

_BY_CODE = {1: ArgumentError, 2: DefinitenessError, 3: SingularityError, 4: SolvabilityError,
            5: NumericError, 6: CudaError}


def check(status: int) -> None:
    """Raise the reference exception class for a non-zero C ABI status."""
    if status == 0:
        return
    from ._lib import lib
    msg = lib.stkg_last_error_message().decode(errors="replace")
    raise _BY_CODE.get(status, StkError)(msg)
