"""Error model of the reference (common.hpp:12-45): morap::Errc codes carried by
morap::Error. Across the C ABI every status is 0 (ok) or 1 + Errc."""
from __future__ import annotations

import enum


class Errc(enum.IntEnum):
    Syntax = 0
    NotCoSafe = 1
    ClosureBlowup = 2
    InvalidDfa = 3
    InvalidModel = 4
    NotRewardFinite = 5
    NonConvergence = 6
    SingularSystem = 7
    DimensionMismatch = 8
    NonSquare = 9
    NotBistochastic = 10
    NoPerfectMatching = 11
    NotPositiveDefinite = 12
    SolverFailure = 13
    DegenerateDirection = 14
    SizeGuard = 15
    CycleGuard = 16
    InvalidConfig = 17
    GenerationFailure = 18
    NoCertificate = 19
    Io = 20


CUDA_ERROR = 100


class MorapError(RuntimeError):
    """morap::Error (common.hpp:36-45); `.code` is the Errc (None for CUDA failures)."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = int(status)
        self.code = Errc(status - 1) if 1 <= status <= 21 else None


def check_status(status: int, msg: str = "") -> None:
    if status != 0:
        raise MorapError(status, msg)
