"""Error taxonomy mirroring the reference (errors.hpp:9-25) + engine codes.

Status codes are those of include/atk.h (`atk_status`); both the CUDA engine
and the CPU oracle report them, and `raise_for_status` turns them into the
same exception classes the reference throws.
"""
from __future__ import annotations


class Error(RuntimeError):
    """atucker::Error — base of every library error."""


class ModeOutOfRange(Error):
    pass


class ShapeMismatch(Error):
    pass


class RankExceedsDim(Error):
    pass


class NotSquare(Error):
    pass


class RankTooLarge(Error):
    pass


class NoConvergence(Error):
    pass


class RankDeficient(Error):
    pass


class NotSPD(Error):
    pass


class ZeroNormInput(Error):
    pass


class EmptyDataset(Error):
    pass


class IoFailure(Error):
    """atucker::IoFailure — .dten / .tucker I/O."""


class FeatureVersionMismatch(Error):
    pass


class SchemaMismatch(Error):
    pass


class CudaError(Error):
    """CUDA runtime failure (also: no B200 visible — there is no CPU fallback)."""


class NcclError(Error):
    pass


class OutOfMemory(Error):
    pass


class InvalidArgument(Error):
    pass


class Unsupported(Error):
    pass


STATUS = {
    1: Error,
    2: ModeOutOfRange,
    3: ShapeMismatch,
    4: RankExceedsDim,
    5: NotSquare,
    6: RankTooLarge,
    7: NoConvergence,
    8: RankDeficient,
    9: NotSPD,
    10: ZeroNormInput,
    11: EmptyDataset,
    12: FeatureVersionMismatch,
    13: SchemaMismatch,
    14: IoFailure,
    20: CudaError,
    21: NcclError,
    22: OutOfMemory,
    23: InvalidArgument,
    24: Unsupported,
}


def raise_for_status(code: int, message: str) -> None:
    if code == 0:
        return
    raise STATUS.get(int(code), Error)(message)
