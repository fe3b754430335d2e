"""Host-side mirror of the reference's `atucker` namespace over the C ABI.

Names, argument meaning and error behaviour follow the reference hot path:
  kernels.hpp  : gram, ttm, ttt_mode
  linalg.hpp   : sym_eig_top_r, thin_qr, spd_solve
  solvers.hpp  : AlsOptions, ModeResult, eig_mode_solver, als_iterate,
                 als_mode_solver, svd_mode_solver
  sthosvd.hpp  : TuckerDecomposition, ModeReport, SthosvdResult, sthosvd,
                 reconstruct, relative_error
  tensor.hpp   : frobenius_norm
Dense tensors are either numpy arrays (host; interpreted column-major, i.e.
`np.asfortranarray`) or `DeviceTensor` handles resident in B200 HBM.  All
compute runs in libatk_cuda.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import Error
from .selector import CostModelParams, SolverKind, Strategy

_DT = {np.dtype(np.float32): _lib.ATK_F32, np.dtype(np.float64): _lib.ATK_F64}
_NP = {_lib.ATK_F32: np.float32, _lib.ATK_F64: np.float64}


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _dims(d) -> C.Array:
    return (C.c_uint64 * len(d))(*[int(v) for v in d])


class Context:
    """One atk_ctx (device, stream, workspace pool, optional NCCL comm)."""

    _default: dict = {}

    def __init__(self, device: int = 0):
        self.lib = _lib.load()
        h = C.c_void_p()
        _lib.check(self.lib.atk_ctx_create(int(device), C.byref(h)))
        self.h = h
        self.device = device

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = cls(device)
        return cls._default[device]

    def set_option(self, key: str, value: float) -> None:
        _lib.check(self.lib.atk_ctx_set_option(self.h, key.encode(), float(value)))

    def set_stream(self, stream_handle: int) -> None:
        _lib.check(self.lib.atk_ctx_set_stream(self.h, C.c_void_p(stream_handle)))

    def synchronize(self) -> None:
        _lib.check(self.lib.atk_ctx_synchronize(self.h))

    @property
    def launch_count(self) -> int:
        return int(self.lib.atk_ctx_launch_count(self.h))

    @staticmethod
    def _nccl_hint() -> None:
        """Point the engine's dlopen at torch's bundled NCCL (same copy as torch.distributed)."""
        import os

        if "ATK_NCCL_PATH" in os.environ:
            return
        try:
            import nvidia.nccl
        except ImportError:
            return
        for d in nvidia.nccl.__path__:
            p = os.path.join(d, "lib", "libnccl.so.2")
            if os.path.exists(p):
                os.environ["ATK_NCCL_PATH"] = p
                return

    def comm_init(self, unique_id: bytes, rank: int, world: int) -> None:
        self._nccl_hint()
        buf = C.create_string_buffer(bytes(unique_id), 128)
        _lib.check(self.lib.atk_comm_init(self.h, buf, int(rank), int(world)))

    def comm_init_host(self, allreduce_f64, broadcast, rank: int, world: int) -> None:
        """Host-staged collectives (atk_comm_init_host): `allreduce_f64(np.ndarray)`
        sums a float64 array in place over the ranks; `broadcast(np.ndarray, root)`
        broadcasts a uint8 array.  Lets several ranks share one GPU."""
        import numpy as np

        def _ar(_user, buf, count):
            try:
                allreduce_f64(np.ctypeslib.as_array(buf, shape=(int(count),)))
                return 0
            except Exception:  # noqa: BLE001 — reported as a status, never across the ABI
                return 1

        def _bc(_user, buf, nbytes, root):
            try:
                if nbytes:
                    a = np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_uint8)), shape=(int(nbytes),))
                    broadcast(a, int(root))
                return 0
            except Exception:  # noqa: BLE001
                return 1

        coll = _lib.HostCollectives(_lib.HOST_ALLREDUCE_FN(_ar), _lib.HOST_BROADCAST_FN(_bc), None)
        self._host_coll = coll  # the C side keeps raw callback pointers
        _lib.check(self.lib.atk_comm_init_host(self.h, C.byref(coll), int(rank), int(world)))

    def comm_stats(self, reset: bool = False) -> dict:
        """Collectives this rank issued (atk_comm_get_stats): counts and payload bytes."""
        buf = (C.c_uint64 * 4)()
        _lib.check(self.lib.atk_comm_get_stats(self.h, C.byref(buf)))
        if reset:
            _lib.check(self.lib.atk_comm_reset_stats(self.h))
        return {"allreduce_calls": buf[0], "allreduce_bytes": buf[1], "gather_calls": buf[2], "gather_bytes": buf[3]}

    @staticmethod
    def nccl_unique_id() -> bytes:
        Context._nccl_hint()
        buf = C.create_string_buffer(128)
        _lib.check(_lib.load().atk_nccl_unique_id(buf))
        return buf.raw

    def close(self) -> None:
        if self.h:
            self.lib.atk_ctx_destroy(self.h)
            self.h = None


def _ctx(ctx: Context | None) -> Context:
    return ctx if ctx is not None else Context.default()


class DeviceTensor:
    """A dense column-major tensor in device memory (atk_tensor handle)."""

    def __init__(self, handle: C.c_void_p, ctx: Context, owner=None):
        self.h = handle
        self.ctx = ctx
        self._owner = owner  # keeps wrapped foreign memory alive
        dt = C.c_int()
        order = C.c_int()
        dims = (C.c_uint64 * _lib.ATK_MAX_ORDER)()
        ptr = C.c_void_p()
        _lib.check(ctx.lib.atk_tensor_info(handle, C.byref(dt), C.byref(order), dims, C.byref(ptr)))
        self.dtype = np.dtype(_NP[dt.value])
        self.dims = tuple(int(dims[m]) for m in range(order.value))
        self.data_ptr = ptr.value

    # -- construction
    @classmethod
    def empty(cls, dims, dtype=np.float64, ctx: Context | None = None) -> "DeviceTensor":
        ctx = _ctx(ctx)
        h = C.c_void_p()
        _lib.check(ctx.lib.atk_tensor_create(ctx.h, _DT[np.dtype(dtype)], len(dims), _dims(dims), C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_numpy(cls, x: np.ndarray, ctx: Context | None = None) -> "DeviceTensor":
        ctx = _ctx(ctx)
        x = np.asfortranarray(x)
        if x.dtype not in _DT:
            raise Error(f"unsupported dtype {x.dtype} (float32 / float64)")
        h = C.c_void_p()
        _lib.check(ctx.lib.atk_tensor_from_host(ctx.h, _DT[x.dtype], x.ndim, _dims(x.shape),
                                                C.c_void_p(x.ctypes.data), C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def wrap(cls, device_ptr: int, dims, dtype, ctx: Context | None = None, owner=None) -> "DeviceTensor":
        """Non-owning view of existing device memory (e.g. a torch CUDA tensor)."""
        ctx = _ctx(ctx)
        h = C.c_void_p()
        _lib.check(ctx.lib.atk_tensor_wrap(ctx.h, _DT[np.dtype(dtype)], len(dims), _dims(dims),
                                           C.c_void_p(device_ptr), C.byref(h)))
        return cls(h, ctx, owner=owner)

    @classmethod
    def uniform(cls, dims, seed: int, dtype=np.float32, ctx: Context | None = None,
                offset: int = 0) -> "DeviceTensor":
        """Counter-hash uniform [-1, 1) generated on the device (bit-exact with the oracle)."""
        t = cls.empty(dims, dtype, ctx)
        _lib.check(t.ctx.lib.atk_fill_uniform(t.ctx.h, t.h, int(seed), int(offset)))
        return t

    # -- access
    @property
    def order(self) -> int:
        return len(self.dims)

    def dim(self, mode: int) -> int:
        return self.dims[mode]

    @property
    def size(self) -> int:
        return int(np.prod(self.dims))

    def to_numpy(self) -> np.ndarray:
        out = np.empty(self.dims, dtype=self.dtype, order="F")
        _lib.check(self.ctx.lib.atk_tensor_to_host(self.ctx.h, self.h, C.c_void_p(out.ctypes.data)))
        return out

    def axpy(self, alpha: float, other: "DeviceTensor") -> None:
        _lib.check(self.ctx.lib.atk_axpy(self.ctx.h, self.h, float(alpha), other.h))

    def free(self) -> None:
        if getattr(self, "h", None):
            self.ctx.lib.atk_tensor_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass

    def __repr__(self) -> str:
        return f"DeviceTensor(dims={self.dims}, dtype={self.dtype})"


def _as_device(x, ctx: Context | None) -> tuple[DeviceTensor, bool]:
    if isinstance(x, DeviceTensor):
        return x, False
    return DeviceTensor.from_numpy(np.asarray(x), ctx), True


def _mat(a, rows_cols=None) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


# ------------------------------------------------------------------ tensor.hpp
def frobenius_norm(x, ctx: Context | None = None) -> float:
    """tensor.hpp:158-168 (fp64 accumulation on the device)."""
    t, tmp = _as_device(x, ctx)
    out = C.c_double()
    _lib.check(t.ctx.lib.atk_frobenius_norm(t.ctx.h, t.h, C.byref(out)))
    if tmp:
        t.free()
    return out.value


# ------------------------------------------------------------------ kernels.hpp
def gram(x, mode: int, ctx: Context | None = None) -> np.ndarray:
    """kernels::gram (kernels.hpp:127-138): X_(n) X_(n)^T, exactly symmetric."""
    t, tmp = _as_device(x, ctx)
    if not (0 <= mode < t.order):
        from .errors import ModeOutOfRange
        raise ModeOutOfRange(f"mode {mode} out of range for order {t.order}")
    n = t.dims[mode]
    s = np.empty((n, n), order="F")
    _lib.check(t.ctx.lib.atk_gram(t.ctx.h, t.h, int(mode), _dptr(s)))
    if tmp:
        t.free()
    return s


def ttm(x, u, mode: int, ctx: Context | None = None):
    """kernels::ttm (kernels.hpp:88-118): Y = X x_n U, U is R x I_n.

    Returns a DeviceTensor when `x` is one, else a numpy array."""
    t, tmp = _as_device(x, ctx)
    u = _mat(u)
    if u.ndim != 2:
        from .errors import ShapeMismatch
        raise ShapeMismatch("ttm matrix must be 2-D")
    h = C.c_void_p()
    _lib.check(t.ctx.lib.atk_ttm(t.ctx.h, t.h, _dptr(u), u.shape[0], u.shape[1], int(mode), C.byref(h)))
    y = DeviceTensor(h, t.ctx)
    if tmp:
        t.free()
        out = y.to_numpy()
        y.free()
        return out
    return y


def ttt_mode(x, y, mode: int, ctx: Context | None = None) -> np.ndarray:
    """kernels::ttt_mode (kernels.hpp:122-124): X_(n) Y_(n)^T."""
    a, ta = _as_device(x, ctx)
    b, tb = _as_device(y, a.ctx)
    if not (0 <= mode < a.order):
        from .errors import ModeOutOfRange
        raise ModeOutOfRange(f"mode {mode} out of range for order {a.order}")
    if not (0 <= mode < b.order):
        from .errors import ModeOutOfRange
        raise ModeOutOfRange(f"mode {mode} out of range for order {b.order}")
    z = np.empty((a.dims[mode], b.dims[mode]), order="F")
    _lib.check(a.ctx.lib.atk_ttt(a.ctx.h, a.h, b.h, int(mode), _dptr(z)))
    if ta:
        a.free()
    if tb:
        b.free()
    return z


# ------------------------------------------------------------------ linalg.hpp
@dataclass
class EigPair:
    values: np.ndarray
    vectors: np.ndarray


@dataclass
class QrPair:
    q: np.ndarray
    r: np.ndarray


def sym_eig_top_r(s, r: int, ctx: Context | None = None) -> EigPair:
    """linalg::sym_eig_top_r (linalg.hpp:101-123)."""
    ctx = _ctx(ctx)
    s = _mat(s)
    if s.ndim != 2 or s.shape[0] != s.shape[1]:
        from .errors import NotSquare
        raise NotSquare("sym_eig_top_r expects a square matrix")
    n = s.shape[0]
    vals = np.empty(max(r, 0))
    vecs = np.empty((n, max(r, 0)), order="F")
    _lib.check(ctx.lib.atk_sym_eig_top_r(ctx.h, _dptr(s), n, int(r), _dptr(vals), _dptr(vecs)))
    return EigPair(vals, vecs)


def thin_qr(a, ctx: Context | None = None) -> QrPair:
    """linalg::thin_qr (linalg.hpp:126-149)."""
    ctx = _ctx(ctx)
    a = _mat(a)
    m, n = a.shape
    q = np.empty((m, n), order="F")
    r = np.empty((n, n), order="F")
    _lib.check(ctx.lib.atk_thin_qr(ctx.h, _dptr(a), m, n, _dptr(q), _dptr(r)))
    return QrPair(q, r)


def spd_solve(a, b, ctx: Context | None = None) -> np.ndarray:
    """linalg::spd_solve (linalg.hpp:169-177)."""
    ctx = _ctx(ctx)
    a = _mat(a)
    b = _mat(b)
    if a.shape[0] != a.shape[1]:
        from .errors import NotSquare
        raise NotSquare("spd_solve expects a square matrix")
    if b.shape[0] != a.shape[0]:
        from .errors import ShapeMismatch
        raise ShapeMismatch("spd_solve right-hand side has wrong row count")
    x = np.empty(b.shape, order="F")
    nrhs = b.shape[1] if b.ndim == 2 else 1
    _lib.check(ctx.lib.atk_spd_solve(ctx.h, _dptr(a), a.shape[0], _dptr(b), nrhs, _dptr(x)))
    return x


# ------------------------------------------------------------------ solvers.hpp
@dataclass
class AlsOptions:
    """solvers.hpp:18-22."""
    num_iters: int = 5
    rel_tol: float = 0.0
    seed: int = 0

    def c(self) -> _lib.AlsOpts:
        return _lib.AlsOpts(int(self.num_iters), float(self.rel_tol), int(self.seed))


@dataclass
class StageTimes:
    gram_ms: float = 0.0
    eig_ms: float = 0.0
    ttm_ms: float = 0.0
    als_ms: float = 0.0
    comm_ms: float = 0.0
    total_ms: float = 0.0

    @classmethod
    def from_c(cls, t: _lib.StageTimes) -> "StageTimes":
        return cls(t.gram_ms, t.eig_ms, t.ttm_ms, t.als_ms, t.comm_ms, t.total_ms)


@dataclass
class ModeResult:
    """solvers.hpp:26-31."""
    factor: np.ndarray
    shrunk: object  # DeviceTensor or numpy array (mirrors the input kind)
    iterations_run: int = 0
    solver_used: SolverKind = SolverKind.Eig
    times: StageTimes = field(default_factory=StageTimes)


def _mode_call(fn_name: str, y, mode: int, r: int, ctx, extra=()) -> ModeResult:
    t, tmp = _as_device(y, ctx)
    if not (0 <= mode < t.order):
        from .errors import ModeOutOfRange
        raise ModeOutOfRange(f"mode {mode} out of range for order {t.order}")
    factor = np.empty((t.dims[mode], max(int(r), 0)), order="F")
    h = C.c_void_p()
    times = _lib.StageTimes()
    return t, tmp, factor, h, times


def _finish(t, tmp, h, factor, times, kind, iters=0) -> ModeResult:
    shrunk = DeviceTensor(h, t.ctx)
    if tmp:
        t.free()
        out = shrunk.to_numpy()
        shrunk.free()
        shrunk = out
    return ModeResult(factor, shrunk, iters, kind, StageTimes.from_c(times))


def eig_mode_solver(y, mode: int, r: int, ctx: Context | None = None) -> ModeResult:
    """eig_mode_solver (solvers.hpp:64-73): gram -> sym_eig_top_r -> ttm."""
    t, tmp, factor, h, times = _mode_call("eig", y, mode, r, ctx)
    _lib.check(t.ctx.lib.atk_eig_mode(t.ctx.h, t.h, int(mode), int(r), _dptr(factor), C.byref(h),
                                      C.byref(times)))
    return _finish(t, tmp, h, factor, times, SolverKind.Eig)


def svd_mode_solver(y, mode: int, r: int, ctx: Context | None = None) -> ModeResult:
    """svd_mode_solver (solvers.hpp:142-162): fp64 on the explicit unfolding (csrc/svd.cu), else the Gram route."""
    t, tmp, factor, h, times = _mode_call("svd", y, mode, r, ctx)
    _lib.check(t.ctx.lib.atk_svd_mode(t.ctx.h, t.h, int(mode), int(r), _dptr(factor), C.byref(h),
                                      C.byref(times)))
    return _finish(t, tmp, h, factor, times, SolverKind.Svd)


def als_mode_solver(y, mode: int, r: int, opts: AlsOptions | None = None, l0=None,
                    ctx: Context | None = None) -> ModeResult:
    """als_mode_solver (solvers.hpp:122-138); L0 from the reference seeding rule unless given."""
    opts = opts or AlsOptions()
    t, tmp, factor, h, times = _mode_call("als", y, mode, r, ctx)
    o = opts.c()
    iters = C.c_int()
    l0p = _dptr(_mat(l0)) if l0 is not None else None
    keep = _mat(l0) if l0 is not None else None
    if keep is not None:
        l0p = _dptr(keep)
    _lib.check(t.ctx.lib.atk_als_mode(t.ctx.h, t.h, int(mode), int(r), C.byref(o), l0p, _dptr(factor),
                                      C.byref(h), C.byref(iters), C.byref(times)))
    return _finish(t, tmp, h, factor, times, SolverKind.Als, iters.value)


@dataclass
class AlsIterateResult:
    """solvers.hpp:79-83."""
    l: np.ndarray
    rfac: object
    iterations_run: int = 0


def als_iterate(y, mode: int, l0, opts: AlsOptions | None = None,
                ctx: Context | None = None) -> AlsIterateResult:
    """als_iterate (solvers.hpp:88-118)."""
    opts = opts or AlsOptions()
    t, tmp = _as_device(y, ctx)
    l0 = _mat(l0)
    if not (0 <= mode < t.order):
        from .errors import ModeOutOfRange
        raise ModeOutOfRange(f"mode {mode} out of range for order {t.order}")
    if l0.shape[0] != t.dims[mode]:
        from .errors import ShapeMismatch
        raise ShapeMismatch(f"initial guess has {l0.shape[0]} rows but mode has dimension {t.dims[mode]}")
    r = l0.shape[1]
    l_out = np.empty((l0.shape[0], r), order="F")
    h = C.c_void_p()
    it = C.c_int()
    o = opts.c()
    _lib.check(t.ctx.lib.atk_als_iterate(t.ctx.h, t.h, int(mode), _dptr(l0), r, C.byref(o), _dptr(l_out),
                                         C.byref(h), C.byref(it)))
    rfac = DeviceTensor(h, t.ctx)
    if tmp:
        t.free()
        out = rfac.to_numpy()
        rfac.free()
        rfac = out
    return AlsIterateResult(l_out, rfac, it.value)


# ------------------------------------------------------------------ sthosvd.hpp
@dataclass
class TuckerDecomposition:
    """sthosvd.hpp:18-22."""
    core: object
    factors: list
    original_dims: tuple


@dataclass
class ModeReport:
    """sthosvd.hpp:25-34 + device per-stage times."""
    mode: int
    solver_used: SolverKind
    selector_decision_time: float
    solver_time: float
    predicted_cost_eig: float
    predicted_cost_als: float
    dims_before: tuple
    dims_after: tuple
    iterations_run: int = 0
    eig_method: str = "jacobi"
    times: StageTimes = field(default_factory=StageTimes)


@dataclass
class SthosvdResult:
    decomposition: TuckerDecomposition
    reports: list


def _selector_callback(strategy: Strategy, opts: AlsOptions):
    params = CostModelParams(opts.num_iters)
    box = {"err": None}

    def cb(_user, mode, i, r, j):
        try:
            return int(strategy.decide(int(mode), int(i), int(r), int(j), params))
        except Exception as e:  # surfaced after the call returns
            box["err"] = e
            return -1

    return _lib.SELECTOR_FN(cb), box


def _reports(reps, order: int) -> list:
    out = []
    for n in range(order):
        rp = reps[n]
        out.append(ModeReport(
            mode=rp.mode, solver_used=SolverKind(rp.solver_used),
            selector_decision_time=rp.selector_decision_time, solver_time=rp.solver_time,
            predicted_cost_eig=rp.predicted_cost_eig, predicted_cost_als=rp.predicted_cost_als,
            dims_before=tuple(int(v) for v in rp.dims_before[:order]),
            dims_after=tuple(int(v) for v in rp.dims_after[:order]),
            iterations_run=rp.iterations_run, eig_method={0: "jacobi", 1: "chfsi", 2: "tridiag", 3: "dense", 4: "svd-jacobi"}.get(rp.eig_method, "?"),
            times=StageTimes.from_c(rp.times)))
    return out


def _split_factors(flat: np.ndarray, dims, ranks) -> list:
    out, off = [], 0
    for i, r in zip(dims, ranks):
        out.append(np.asfortranarray(flat[off:off + i * r].reshape((i, r), order="F")))
        off += i * r
    return out


def sthosvd(x, ranks, strategy: Strategy | None = None, opts: AlsOptions | None = None,
            ctx: Context | None = None, global_dims=None) -> SthosvdResult:
    """sthosvd (sthosvd.hpp:126-194).

    `x` may be a numpy array (host: copied in, core copied back) or a
    DeviceTensor (core stays on the device).  Under a multi-GPU context `x`
    is this rank's slab of the last mode and `global_dims` the full shape."""
    strategy = strategy or Strategy.fixed_eig()
    opts = opts or AlsOptions()
    t, tmp = _as_device(x, ctx)
    order = t.order
    ranks = [int(r) for r in ranks]
    if len(ranks) != order:
        from .errors import RankExceedsDim
        raise RankExceedsDim(f"expected {order} truncations, got {len(ranks)}")
    if strategy.kind is Strategy.Kind.Manual and len(strategy.choices) != order:
        raise Error(f"manual strategy must choose a solver for each of the {order} modes")
    gdims = tuple(global_dims) if global_dims is not None else t.dims
    factors = np.empty(sum(i * r for i, r in zip(gdims, ranks)))
    reps = (_lib.ModeReportC * order)()
    cb, box = _selector_callback(strategy, opts)
    o = opts.c()
    h = C.c_void_p()
    code = t.ctx.lib.atk_sthosvd(t.ctx.h, t.h, _dims(ranks), cb, None, C.byref(o), C.byref(h),
                                 _dptr(factors), reps)
    if box["err"] is not None:
        raise box["err"]
    try:
        _lib.check(code)
    finally:
        if tmp:
            t.free()
    core = DeviceTensor(h, t.ctx)
    if tmp:
        c = core.to_numpy()
        core.free()
        core = c
    dec = TuckerDecomposition(core, _split_factors(factors, gdims, ranks), gdims)
    return SthosvdResult(dec, _reports(reps, order))


def sthosvd_host(x: np.ndarray, ranks, strategy: Strategy | None = None,
                 opts: AlsOptions | None = None, ctx: Context | None = None) -> SthosvdResult:
    """The e2e host-buffer entry (atk_sthosvd_host): H2D, st-HOSVD, D2H of the core."""
    ctx = _ctx(ctx)
    strategy = strategy or Strategy.fixed_eig()
    opts = opts or AlsOptions()
    if not (x.flags.f_contiguous or x.ndim == 1):
        x = np.asfortranarray(x)
    order = x.ndim
    ranks = [int(r) for r in ranks]
    core = np.empty(ranks, dtype=x.dtype, order="F")
    factors = np.empty(sum(i * r for i, r in zip(x.shape, ranks)))
    reps = (_lib.ModeReportC * order)()
    cb, box = _selector_callback(strategy, opts)
    o = opts.c()
    code = ctx.lib.atk_sthosvd_host(ctx.h, _DT[x.dtype], order, _dims(x.shape), C.c_void_p(x.ctypes.data),
                                    _dims(ranks), cb, None, C.byref(o), C.c_void_p(core.ctypes.data),
                                    _dptr(factors), reps)
    if box["err"] is not None:
        raise box["err"]
    _lib.check(code)
    dec = TuckerDecomposition(core, _split_factors(factors, x.shape, ranks), tuple(x.shape))
    return SthosvdResult(dec, _reports(reps, order))


def _flat_factors(t: TuckerDecomposition) -> np.ndarray:
    return np.concatenate([np.asarray(f, dtype=np.float64).ravel(order="F") for f in t.factors])


def reconstruct(t: TuckerDecomposition, ctx: Context | None = None):
    """reconstruct (sthosvd.hpp:197-209)."""
    core, tmp = _as_device(t.core, ctx)
    order = core.order
    if len(t.factors) != order or len(t.original_dims) != order:
        from .errors import ShapeMismatch
        raise ShapeMismatch("decomposition has inconsistent order")
    for n in range(order):
        f = np.asarray(t.factors[n])
        if f.shape[0] != t.original_dims[n] or f.shape[1] != core.dims[n]:
            from .errors import ShapeMismatch
            raise ShapeMismatch(f"factor {n + 1} does not match the core and original dims")
    flat = _flat_factors(t)
    h = C.c_void_p()
    _lib.check(core.ctx.lib.atk_reconstruct(core.ctx.h, core.h, _dptr(flat), _dims(t.original_dims),
                                            C.byref(h)))
    y = DeviceTensor(h, core.ctx)
    if tmp:
        core.free()
        out = y.to_numpy()
        y.free()
        return out
    return y


def relative_error(x, t: TuckerDecomposition, ctx: Context | None = None) -> float:
    """relative_error (sthosvd.hpp:212-223)."""
    xd, tx = _as_device(x, ctx)
    core = t.core
    tc = False
    if not isinstance(core, DeviceTensor):
        core = DeviceTensor.from_numpy(np.asarray(core, dtype=xd.dtype), xd.ctx)
        tc = True
    flat = _flat_factors(t)
    out = C.c_double()
    try:
        _lib.check(xd.ctx.lib.atk_relative_error(xd.ctx.h, xd.h, core.h, _dptr(flat), C.byref(out)))
    finally:
        if tx:
            xd.free()
        if tc:
            core.free()
    return out.value


# ------------------------------------------------------------------ instrumentation.hpp
def reset_gemm_counters() -> None:
    _lib.load().atk_reset_gemm_counters()


class AllocScope:
    """instr::AllocScope (instrumentation.hpp:144-150): tracks live device tensor
    payloads while the `with` block runs; `watch_elems` = the size to count
    (the input's) in live/peak_watched.  `stats()` mirrors AllocTracker::Stats."""

    def __init__(self, watch_elems: int):
        self.watch = int(watch_elems)

    def __enter__(self) -> "AllocScope":
        _lib.load().atk_alloc_tracking_enable(self.watch)
        return self

    def __exit__(self, *exc) -> None:
        _lib.load().atk_alloc_tracking_disable()

    def stats(self) -> dict:
        st = _lib.AllocStats()
        _lib.check(_lib.load().atk_alloc_tracking_stats(C.byref(st)))
        return {k: int(getattr(st, k)) for k, _ in _lib.AllocStats._fields_}


def gemm_calls() -> int:
    return int(_lib.load().atk_gemm_calls())


def gemm_flops() -> int:
    return int(_lib.load().atk_gemm_flops())
