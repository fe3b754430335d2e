"""The solver-selector hook: Strategy + cost model + decision-tree predict.

Mirrors sthosvd.hpp:39-107 (Strategy::decide) and selector.hpp:27-104
(extract_features, f_eig/f_qr/f_inv, cost_eig/cost_als, heuristic_choice,
predict).  The offline CART trainer (selector.hpp:164-328) is out of scope.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field

from .errors import Error, FeatureVersionMismatch, SchemaMismatch

FEATURE_ORDER_VERSION = 1
FEATURE_NAMES = ("I_n", "R_n", "J_n", "I_n^2", "R_n^2", "I_n*R_n", "R_n^2/I_n", "R_n^2/J_n",
                 "I_n/J_n", "R_n/J_n")


class SolverKind(enum.IntEnum):
    """solver_kind.hpp:11 — label encoding 0 = EIG, 1 = ALS, 2 = SVD."""
    Eig = 0
    Als = 1
    Svd = 2

    def __str__(self) -> str:  # solver_kind.hpp:13-20
        return self.name.lower()


def solver_kind_from_string(s: str) -> SolverKind:
    """solver_kind.hpp:22-27."""
    t = {"eig": SolverKind.Eig, "EIG": SolverKind.Eig, "als": SolverKind.Als,
         "ALS": SolverKind.Als, "svd": SolverKind.Svd, "SVD": SolverKind.Svd}
    if s not in t:
        raise Error(f"unknown solver name: {s}")
    return t[s]


def extract_features(i: float, r: float, j: float) -> tuple:
    """selector.hpp:27-29."""
    return (i, r, j, i * i, r * r, i * r, r * r / i, r * r / j, i / j, r / j)


@dataclass
class CostModelParams:
    num_iters: int = 5


def f_eig(i: float) -> float:
    return 9.0 * i * i * i


def f_qr(i: float, r: float) -> float:
    return 2.0 * i * r * r - (2.0 / 3.0) * r * r * r


def f_inv(r: float) -> float:
    return 2.0 * r * r * r


def cost_eig(i: float, r: float, j: float, params: CostModelParams | None = None) -> float:
    """selector.hpp:41-43."""
    return i * i * j + 2.0 * i * r * j + f_eig(i)


def cost_als(i: float, r: float, j: float, params: CostModelParams | None = None) -> float:
    """selector.hpp:46-52."""
    n = (params or CostModelParams()).num_iters
    per_iter = (2.0 * i * j * r + 2.0 * j * r * r + 2.0 * i * j * r + 2.0 * j * r * r
                + 4.0 * i * r * r + 2.0 * f_inv(r))
    return per_iter * n + 2.0 * j * r * r + f_qr(i, r)


def heuristic_choice(i: float, r: float, j: float, params: CostModelParams | None = None) -> SolverKind:
    """selector.hpp:55-58 — ties go to EIG."""
    return SolverKind.Eig if cost_eig(i, r, j, params) <= cost_als(i, r, j, params) else SolverKind.Als


@dataclass
class Node:
    leaf: bool = False
    feature_index: int = -1
    threshold: float = 0.0
    left: int = -1
    right: int = -1
    label: int = 0


@dataclass
class DecisionTreeModel:
    """selector.hpp:62-84 (the fields predict needs)."""
    nodes: list = field(default_factory=list)
    root: int = -1
    feature_order_version: int = FEATURE_ORDER_VERSION


def predict(model: DecisionTreeModel, f: tuple) -> SolverKind:
    """selector.hpp:88-104 — deterministic root-to-leaf descent."""
    if model.feature_order_version != FEATURE_ORDER_VERSION:
        raise FeatureVersionMismatch(
            f"model was trained with feature order version {model.feature_order_version}")
    if model.root < 0 or model.root >= len(model.nodes):
        raise SchemaMismatch("decision tree has no valid root")
    nid = model.root
    for _ in range(len(model.nodes) + 1):
        node = model.nodes[nid]
        if node.leaf:
            return SolverKind.Eig if node.label == 0 else SolverKind.Als
        nid = node.left if f[node.feature_index] <= node.threshold else node.right
        if nid < 0 or nid >= len(model.nodes):
            raise SchemaMismatch("decision tree child id out of range")
    raise SchemaMismatch("decision tree descent did not reach a leaf")


class Strategy:
    """sthosvd.hpp:39-107 — how the driver picks the per-mode solver."""

    class Kind(enum.Enum):
        Adaptive = "adaptive"
        CostModel = "costmodel"
        FixedEig = "eig"
        FixedAls = "als"
        FixedSvd = "svd"
        Manual = "manual"
        Roofline = "roofline"

    def __init__(self, kind: "Strategy.Kind", choices=None, model: DecisionTreeModel | None = None,
                 roofline=None):
        self.kind = kind
        self.choices = list(choices or [])
        self.model = model
        self.roofline_params = roofline

    @staticmethod
    def adaptive(model: DecisionTreeModel) -> "Strategy":
        return Strategy(Strategy.Kind.Adaptive, model=model)

    @staticmethod
    def cost_model() -> "Strategy":
        return Strategy(Strategy.Kind.CostModel)

    @staticmethod
    def roofline(dtype: str = "f32", num_iters: int = 5, **overrides) -> "Strategy":
        """B200 roofline cost model (atk_roofline_selector):
        each stage costs max(flops / peak, bytes / HBM bandwidth) plus measured
        fixed costs; EIG iff its modelled time <= ALS's.  `overrides` set fields
        of atk_roofline_params (hbm_gbs, tf32_tflops, fp64_tflops, eig_small_ms,
        eig_large_ms, als_iter_overhead_ms)."""
        from . import _lib

        p = _lib.RooflineParams()
        _lib.load().atk_roofline_params_default(p, 0 if dtype in ("f32", "float32") else 1, int(num_iters))
        for k, v in overrides.items():
            if not hasattr(p, k):
                raise Error(f"unknown roofline parameter '{k}'")
            setattr(p, k, v)
        return Strategy(Strategy.Kind.Roofline, roofline=p)

    def roofline_times(self, i: int, r: int, j: int, mode: int | None = None) -> tuple:
        """(EIG seconds, ALS seconds) under the roofline model (with `mode`, the
        one-pass ALS of mode 0 is priced as such)."""
        import ctypes as C

        from . import _lib

        lib, p = _lib.load(), C.byref(self.roofline_params)
        als = (lib.atk_roofline_time_als(p, float(i), float(r), float(j)) if mode is None else
               lib.atk_roofline_time_als_mode(p, int(mode), float(i), float(r), float(j)))
        return lib.atk_roofline_time_eig(p, float(i), float(r), float(j)), als

    @staticmethod
    def fixed_eig() -> "Strategy":
        return Strategy(Strategy.Kind.FixedEig)

    @staticmethod
    def fixed_als() -> "Strategy":
        return Strategy(Strategy.Kind.FixedAls)

    @staticmethod
    def fixed_svd() -> "Strategy":
        return Strategy(Strategy.Kind.FixedSvd)

    @staticmethod
    def manual(choices) -> "Strategy":
        ch = [SolverKind(c) if not isinstance(c, str) else solver_kind_from_string(
            {"e": "eig", "a": "als"}.get(c, c)) for c in choices]
        if any(c == SolverKind.Svd for c in ch):
            raise Error("manual strategies choose between eig and als")
        return Strategy(Strategy.Kind.Manual, choices=ch)

    @staticmethod
    def parse(spec: str) -> "Strategy":
        """CLI spelling (atucker.cpp:58-97): adaptive|costmodel|eig|als|svd|manual:e,a,..."""
        if spec.startswith("manual:"):
            return Strategy.manual(spec[len("manual:"):].split(","))
        table = {"costmodel": Strategy.cost_model, "eig": Strategy.fixed_eig,
                 "als": Strategy.fixed_als, "svd": Strategy.fixed_svd, "roofline": Strategy.roofline}
        if spec not in table:
            raise Error(f"unknown strategy '{spec}'")
        return table[spec]()

    def decide(self, mode: int, i: int, r: int, j: int,
               params: CostModelParams | None = None) -> SolverKind:
        k = self.kind
        if k is Strategy.Kind.Adaptive:
            return predict(self.model, extract_features(float(i), float(r), float(j)))
        if k is Strategy.Kind.CostModel:
            return heuristic_choice(float(i), float(r), float(j), params)
        if k is Strategy.Kind.Roofline:
            import ctypes as C

            from . import _lib

            return SolverKind(_lib.load().atk_roofline_selector(C.cast(C.pointer(self.roofline_params), C.c_void_p),
                                                                 int(mode), int(i), int(r), int(j)))
        if k is Strategy.Kind.FixedEig:
            return SolverKind.Eig
        if k is Strategy.Kind.FixedAls:
            return SolverKind.Als
        if k is Strategy.Kind.FixedSvd:
            return SolverKind.Svd
        return self.choices[mode]

    def name(self) -> str:
        if self.kind is Strategy.Kind.Manual:
            return "manual:" + ",".join("e" if c == SolverKind.Eig else "a" for c in self.choices)
        return self.kind.value
