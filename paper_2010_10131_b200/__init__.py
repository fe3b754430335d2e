"""B200-native a-Tucker st-HOSVD engine (drop-in for the reference hot path).

The compute lives in libatk_cuda.so (hand-written sm_100a CUDA behind the C
ABI of include/atk.h); this package is the host-side mirror of the
reference's `atucker` namespace (sthosvd.hpp / solvers.hpp / kernels.hpp /
linalg.hpp / selector.hpp).
"""
from .errors import (CudaError, Error, ModeOutOfRange, NcclError, NoConvergence, NotSPD, NotSquare,
                     OutOfMemory, RankDeficient, RankExceedsDim, RankTooLarge, ShapeMismatch,
                     Unsupported, ZeroNormInput)
from .selector import (CostModelParams, DecisionTreeModel, Node, SolverKind, Strategy, cost_als,
                       cost_eig, extract_features, heuristic_choice, predict)

__all__ = [
    "Error", "ModeOutOfRange", "ShapeMismatch", "RankExceedsDim", "NotSquare", "RankTooLarge",
    "NoConvergence", "RankDeficient", "NotSPD", "ZeroNormInput", "CudaError", "NcclError",
    "OutOfMemory", "Unsupported", "SolverKind", "Strategy", "CostModelParams",
    "DecisionTreeModel", "Node", "cost_eig", "cost_als", "heuristic_choice", "extract_features",
    "predict",
]


_SUBMODULES = {"atucker", "build", "dist", "errors", "selector", "tensor_io"}


def __getattr__(name):
    # The CUDA-backed API is imported lazily so that CPU-only tooling (tests of
    # the selector / oracle / ABI surface) can import the package without a GPU.
    import importlib

    if name.startswith("_") or name in _SUBMODULES:
        raise AttributeError(name)  # lets `from pkg import submodule` import it
    atucker = importlib.import_module(".atucker", __name__)
    if hasattr(atucker, name):
        return getattr(atucker, name)
    raise AttributeError(name)
