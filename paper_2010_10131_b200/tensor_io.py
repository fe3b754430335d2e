"""The reference's file formats: .dten tensors (tensor_io.hpp:15-99) and the
.tucker output directory (tucker_io.hpp:20-74).  SURVEY §8(f) row 3.

Large tensors go through the engine: `read_dten_device` / `write_dten` on a
DeviceTensor stream the f64 payload between the file and HBM in
double-buffered pinned chunks (csrc/dten_io.cu), narrowing to fp32 on the
device when asked.  Small host arrays (factors, cores, test fixtures) use the
host mirror below, byte-identical to the reference's writer (checked against
files written by the reference's own write_dten, tests/golden/ref_*.dten).
Every failure raises the reference's IoFailure with read_dten's messages.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import struct
from pathlib import Path

import numpy as np

from .errors import IoFailure

_MAGIC = b"DTEN"
_VERSION = 1


# ------------------------------------------------------------------ host mirror
def write_dten(path, x) -> None:
    """write_dten (tensor_io.hpp:39-52).  A DeviceTensor is streamed by the
    engine; a numpy array (or DenseMatrix-like 2-D array) is written here."""
    from . import atucker

    if isinstance(x, atucker.DeviceTensor):
        atucker._lib.check(x.ctx.lib.atk_tensor_write_dten(x.ctx.h, x.h, os.fsencode(str(path))))
        return
    a = np.asarray(x, dtype=np.float64)
    if a.ndim == 0:
        raise IoFailure("cannot write an order-0 tensor")
    try:
        with open(path, "wb") as f:
            f.write(_MAGIC + struct.pack("<II", _VERSION, a.ndim) + struct.pack(f"<{a.ndim}Q", *a.shape))
            f.write(np.asfortranarray(a).astype("<f8", copy=False).tobytes(order="F"))
    except OSError as e:
        raise IoFailure(f"cannot open {path} for writing: {e}") from None


def _header(f, path):
    if f.read(4) != _MAGIC:
        raise IoFailure(f"{path}: not a .dten file (bad magic)")
    b = f.read(4)
    version = struct.unpack("<I", b)[0] if len(b) == 4 else 0
    if version != _VERSION:
        raise IoFailure(f"{path}: unsupported .dten version {version}")
    b = f.read(4)
    order = struct.unpack("<I", b)[0] if len(b) == 4 else 0
    if order == 0:
        raise IoFailure(f"{path}: truncated or empty header")
    b = f.read(8 * order)
    if len(b) != 8 * order:
        raise IoFailure(f"{path}: truncated dims block")
    dims = struct.unpack(f"<{order}Q", b)
    total = 1
    for d in dims:
        if d == 0:
            raise IoFailure(f"{path}: zero dimension in header")
        if d > (1 << 40) // total:
            raise IoFailure(f"{path}: dims product is implausibly large")
        total *= d
    return dims, total


def read_dten(path) -> np.ndarray:
    """read_dten (tensor_io.hpp:62-91) into a host fp64 array (column-major)."""
    try:
        f = open(path, "rb")
    except OSError:
        raise IoFailure(f"cannot open {path}") from None
    with f:
        dims, total = _header(f, path)
        raw = f.read(8 * total)
    if len(raw) != 8 * total:
        raise IoFailure(f"{path}: truncated payload, expected {8 * total} bytes but read {len(raw)}")
    return np.frombuffer(raw, dtype="<f8").reshape(dims, order="F").astype(np.float64)


def read_dten_matrix(path) -> np.ndarray:
    """read_dten_matrix (tensor_io.hpp:93-97)."""
    t = read_dten(path)
    if t.ndim != 2:
        raise IoFailure(f"{path}: expected an order-2 .dten")
    return t


def dten_info(path) -> tuple:
    """Header only (the engine's parser; CPU-only, no GPU needed)."""
    from . import _lib

    order = C.c_int()
    dims = (C.c_uint64 * _lib.ATK_MAX_ORDER)()
    _lib.check(_lib.load().atk_dten_info(os.fsencode(str(path)), C.byref(order), dims))
    return tuple(int(dims[m]) for m in range(order.value))


# ------------------------------------------------------------------ engine (device) path
def read_dten_device(path, dtype=np.float32, ctx=None):
    """Stream a .dten file into a new DeviceTensor of `dtype` (f32 or f64)."""
    from . import atucker

    ctx = atucker._ctx(ctx)
    h = C.c_void_p()
    dt = atucker._DT[np.dtype(dtype)]
    atucker._lib.check(ctx.lib.atk_tensor_read_dten(ctx.h, os.fsencode(str(path)), dt, C.byref(h)))
    return atucker.DeviceTensor(h, ctx)


# ------------------------------------------------------------------ .tucker directory
def _report_json(r) -> dict:
    """mode_report_to_json (tucker_io.hpp:20-30): 1-based modes."""
    return {"mode": int(r.mode) + 1, "solver": str(r.solver_used),
            "selector_decision_time_s": float(r.selector_decision_time),
            "solver_time_s": float(r.solver_time),
            "predicted_cost_eig": float(r.predicted_cost_eig),
            "predicted_cost_als": float(r.predicted_cost_als),
            "dims_before": [int(d) for d in r.dims_before], "dims_after": [int(d) for d in r.dims_after]}


def save_tucker(directory, t, reports=(), strategy_name: str = "eig", seed: int = 0) -> None:
    """save_tucker (tucker_io.hpp:32-60): core.dten, factor_<n>.dten (1-based,
    order-2), meta.json (keys sorted, as nlohmann::json dumps them)."""
    d = Path(directory)
    try:
        d.mkdir(parents=True, exist_ok=True)
    except OSError as e:
        raise IoFailure(f"cannot create directory {directory}: {e}") from None
    write_dten(d / "core.dten", t.core)
    ranks = []
    for n, fac in enumerate(t.factors):
        write_dten(d / f"factor_{n + 1}.dten", np.asarray(fac))
        ranks.append(int(np.asarray(fac).shape[1]))
    meta = {"schema_version": 1, "original_dims": [int(x) for x in t.original_dims], "ranks": ranks,
            "strategy": strategy_name, "seed": int(seed), "reports": [_report_json(r) for r in reports]}
    try:
        (d / "meta.json").write_text(json.dumps(meta, indent=2, sort_keys=True) + "\n")
    except OSError as e:
        raise IoFailure(f"failed writing {directory}/meta.json: {e}") from None


def load_tucker(directory):
    """load_tucker (tucker_io.hpp:62-74): host core + factors."""
    from .atucker import TuckerDecomposition

    d = Path(directory)
    if not d.is_dir():
        raise IoFailure(f"{directory} is not a .tucker directory")
    core = read_dten(d / "core.dten")
    factors, odims = [], []
    for n in range(core.ndim):
        f = read_dten_matrix(d / f"factor_{n + 1}.dten")
        if f.shape[1] != core.shape[n]:
            raise IoFailure(f"{directory}: factor {n + 1} does not match the core dimensions")
        factors.append(np.asfortranarray(f))
        odims.append(f.shape[0])
    return TuckerDecomposition(core, factors, tuple(odims))
