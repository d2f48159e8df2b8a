"""Error taxonomy of the hot path — the reference's ``sdpsim::Errc`` / ``Error``
(errors.hpp:8-49) plus the GPU-side ``CudaError``.  ``str(err)`` is the
reference's ``"<Errc>: detail"`` message."""
from __future__ import annotations

import enum


class Errc(enum.IntEnum):
    OutOfRange = 1
    NonDivisible = 2
    Infeasible = 3
    SizeMismatch = 4
    TypeMismatch = 5
    ShapeError = 6
    BoundaryViolation = 7
    EmptyProfile = 8
    ConfigError = 9
    CudaError = 10


class Error(RuntimeError):
    """sdpsim::Error: carries the error code; what() is "<Errc>: detail"."""

    def __init__(self, code, what: str = ""):
        self.code = Errc(int(code))
        if not what.startswith(self.code.name + ":"):
            what = f"{self.code.name}: {what}"
        super().__init__(what)


def raise_error(code: Errc, what: str):
    """sdpsim::raise (errors.hpp:32-34)."""
    raise Error(code, f"{Errc(code).name}: {what}")
