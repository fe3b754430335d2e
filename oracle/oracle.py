"""ctypes front-end of the CPU oracle (oracle/atk_oracle.cpp).

TEST INFRASTRUCTURE ONLY — imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, as the *checker*.  The
product package never imports it.

Every function mirrors the reference symbol of the same name (see the C++
file for file:line citations) and takes/returns float64 numpy arrays in
column-major (Fortran) order.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"

_dp = C.POINTER(C.c_double)
_up = C.POINTER(C.c_uint64)
SELECTOR_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64)

_lib = None


def blas_path() -> str:
    import scipy

    libs = Path(scipy.__file__).resolve().parent.parent / "scipy.libs"
    cands = sorted(libs.glob("libscipy_openblas-*.so"))
    if not cands:
        raise RuntimeError("scipy's bundled OpenBLAS not found")
    return str(cands[0])


def build() -> Path:
    if not LIB.exists() or LIB.stat().st_mtime < (HERE / "atk_oracle.cpp").stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE), "liboracle.so"], check=True, capture_output=True)
    return LIB


def load() -> C.CDLL:
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(str(LIB))
        lib.or_last_error.restype = C.c_char_p
        lib.or_init.argtypes = [C.c_char_p]
        lib.or_mix_seed.restype = C.c_uint64
        lib.or_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.or_frobenius_norm.restype = C.c_double
        lib.or_frobenius_norm.argtypes = [_dp, C.c_uint64]
        lib.or_cost_eig.restype = C.c_double
        lib.or_cost_eig.argtypes = [C.c_double] * 3
        lib.or_cost_als.restype = C.c_double
        lib.or_cost_als.argtypes = [C.c_double] * 3 + [C.c_int]
        lib.or_gemm_calls.restype = C.c_longlong
        lib.or_gemm_flops.restype = C.c_longlong
        lib.or_set_threads.argtypes = [C.c_int]
        lib.or_hash_uniform.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_float)]
        lib.or_sthosvd.argtypes = [_dp, _up, C.c_int, _up, SELECTOR_FN, C.c_void_p, C.c_int, C.c_double,
                                   C.c_uint64, _dp, _dp, _dp]
        lib.or_als_mode.argtypes = [_dp, _up, C.c_int, C.c_int, C.c_uint64, C.c_int, C.c_double,
                                    C.c_uint64, _dp, _dp, C.POINTER(C.c_int)]
        lib.or_als_iterate.argtypes = [_dp, _up, C.c_int, C.c_int, _dp, C.c_uint64, C.c_int, C.c_double,
                                       _dp, _dp, C.POINTER(C.c_int), _dp]
        code = lib.or_init(blas_path().encode())
        if code:
            raise RuntimeError(lib.or_last_error().decode())
        _lib = lib
    return _lib


def _check(code: int) -> None:
    if code:
        from paper_2010_10131_b200.errors import raise_for_status

        raise_for_status(code, load().or_last_error().decode())


def _f(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _d(dims):
    return (C.c_uint64 * len(dims))(*[int(v) for v in dims])


def set_threads(n: int) -> None:
    load().or_set_threads(int(n))


# ------------------------------------------------------------------ tensor.hpp
def mix_seed(seed: int, salt: int) -> int:
    return int(load().or_mix_seed(seed, salt))


def random_tensor(dims, seed: int, dist: str = "uniform01") -> np.ndarray:
    out = np.empty(dims, order="F")
    _check(load().or_random_tensor(_d(dims), len(dims), C.c_uint64(seed), 0 if dist == "uniform01" else 1,
                                   _p(out)))
    return out


def hash_uniform(seed: int, n: int, start: int = 0) -> np.ndarray:
    out = np.empty(n, dtype=np.float32)
    load().or_hash_uniform(C.c_uint64(seed), C.c_uint64(start), C.c_uint64(n),
                           out.ctypes.data_as(C.POINTER(C.c_float)))
    return out


def als_initial_guess(rows: int, r: int, seed: int, mode: int) -> np.ndarray:
    out = np.empty((rows, r), order="F")
    _check(load().or_als_initial_guess(C.c_uint64(rows), C.c_uint64(r), C.c_uint64(seed),
                                       C.c_uint64(mode), _p(out)))
    return out


def frobenius_norm(x) -> float:
    x = _f(x)
    return float(load().or_frobenius_norm(_p(x), x.size))


def matricize(x, mode: int) -> np.ndarray:
    x = _f(x)
    n = x.shape[mode]
    out = np.empty((n, x.size // n), order="F")
    _check(load().or_matricize(_p(x), _d(x.shape), x.ndim, int(mode), _p(out)))
    return out


# ------------------------------------------------------------------ kernels.hpp
def gram(x, mode: int) -> np.ndarray:
    x = _f(x)
    if not 0 <= mode < x.ndim:
        from paper_2010_10131_b200.errors import ModeOutOfRange

        raise ModeOutOfRange(f"mode {mode} out of range for order {x.ndim}")
    n = x.shape[mode]
    out = np.empty((n, n), order="F")
    _check(load().or_gram(_p(x), _d(x.shape), x.ndim, int(mode), _p(out)))
    return out


def ttm(x, u, mode: int) -> np.ndarray:
    x, u = _f(x), _f(u)
    dims = list(x.shape)
    if 0 <= mode < x.ndim:
        dims[mode] = u.shape[0]
    out = np.empty(dims, order="F")
    _check(load().or_ttm(_p(x), _d(x.shape), x.ndim, _p(u), u.shape[0], u.shape[1], int(mode), _p(out)))
    return out


def ttt_mode(x, y, mode: int) -> np.ndarray:
    x, y = _f(x), _f(y)
    out = np.empty((x.shape[mode], y.shape[mode]), order="F")
    _check(load().or_ttt(_p(x), _d(x.shape), _p(y), _d(y.shape), x.ndim, int(mode), _p(out)))
    return out


# ------------------------------------------------------------------ linalg.hpp
@dataclass
class EigPair:
    values: np.ndarray
    vectors: np.ndarray


def sym_eig_top_r(s, r: int) -> EigPair:
    s = _f(s)
    rows, cols = s.shape
    vals = np.empty(max(r, 0))
    vecs = np.empty((rows, max(r, 0)), order="F")
    _check(load().or_sym_eig_top_r(_p(s), rows, cols, C.c_uint64(r), _p(vals), _p(vecs)))
    return EigPair(vals, vecs)


def thin_qr(a):
    a = _f(a)
    m, n = a.shape
    q, r = np.empty((m, n), order="F"), np.empty((n, n), order="F")
    _check(load().or_thin_qr(_p(a), m, n, _p(q), _p(r)))
    return q, r


def thin_svd(a):
    a = _f(a)
    m, n = a.shape
    k = min(m, n)
    u, s, vt = np.empty((m, k), order="F"), np.empty(k), np.empty((k, n), order="F")
    _check(load().or_thin_svd(_p(a), m, n, _p(u), _p(s), _p(vt)))
    return u, s, vt


def spd_solve(a, b) -> np.ndarray:
    a, b = _f(a), _f(b)
    if b.ndim == 1:
        b = b.reshape(-1, 1, order="F")
    x = np.empty(b.shape, order="F")
    _check(load().or_spd_solve(_p(a), a.shape[0], _p(b), b.shape[1], _p(x)))
    return x


def gemm(a, b, trans_a=False, trans_b=False) -> np.ndarray:
    a, b = _f(a), _f(b)
    m = a.shape[1] if trans_a else a.shape[0]
    n = b.shape[0] if trans_b else b.shape[1]
    c = np.empty((m, n), order="F")
    _check(load().or_gemm(_p(a), a.shape[0], a.shape[1], _p(b), b.shape[0], b.shape[1], int(trans_a),
                          int(trans_b), _p(c)))
    return c


# ------------------------------------------------------------------ solvers.hpp
@dataclass
class ModeResult:
    factor: np.ndarray
    shrunk: np.ndarray
    iterations_run: int = 0


def _check_mode(x, mode):
    if not 0 <= mode < x.ndim:
        from paper_2010_10131_b200.errors import ModeOutOfRange

        raise ModeOutOfRange(f"mode {mode} out of range for order {x.ndim}")


def _shrunk_dims(x, mode, r):
    _check_mode(x, mode)
    d = list(x.shape)
    d[mode] = r
    return d


def eig_mode_solver(y, mode: int, r: int) -> ModeResult:
    y = _f(y)
    _check_mode(y, mode)
    f = np.empty((y.shape[mode], r), order="F")
    s = np.empty(_shrunk_dims(y, mode, r), order="F")
    _check(load().or_eig_mode(_p(y), _d(y.shape), y.ndim, int(mode), C.c_uint64(r), _p(f), _p(s)))
    return ModeResult(f, s)


def svd_mode_solver(y, mode: int, r: int) -> ModeResult:
    y = _f(y)
    _check_mode(y, mode)
    f = np.empty((y.shape[mode], r), order="F")
    s = np.empty(_shrunk_dims(y, mode, r), order="F")
    _check(load().or_svd_mode(_p(y), _d(y.shape), y.ndim, int(mode), C.c_uint64(r), _p(f), _p(s)))
    return ModeResult(f, s)


def als_mode_solver(y, mode: int, r: int, num_iters=5, rel_tol=0.0, seed=0) -> ModeResult:
    y = _f(y)
    _check_mode(y, mode)
    f = np.empty((y.shape[mode], r), order="F")
    s = np.empty(_shrunk_dims(y, mode, r), order="F")
    it = C.c_int()
    _check(load().or_als_mode(_p(y), _d(y.shape), y.ndim, int(mode), r, int(num_iters), float(rel_tol),
                              int(seed), _p(f), _p(s), C.byref(it)))
    return ModeResult(f, s, it.value)


def als_iterate(y, mode: int, l0, num_iters=5, rel_tol=0.0, history=False):
    y, l0 = _f(y), _f(l0)
    r = l0.shape[1]
    l_out = np.empty(l0.shape, order="F")
    rfac = np.empty(_shrunk_dims(y, mode, r), order="F")
    it = C.c_int()
    hist = np.empty((num_iters,) + l0.shape) if history else None
    _check(load().or_als_iterate(_p(y), _d(y.shape), y.ndim, int(mode), _p(l0), r, int(num_iters),
                                 float(rel_tol), _p(l_out), _p(rfac), C.byref(it),
                                 _p(hist) if history else None))
    return l_out, rfac, it.value, (hist[: it.value] if history else None)


# ------------------------------------------------------------------ sthosvd.hpp
@dataclass
class SthosvdResult:
    core: np.ndarray
    factors: list
    reports: np.ndarray  # order x {solver, decide_s, solve_s, cost_eig, cost_als}


def sthosvd(x, ranks, decide=None, num_iters=5, rel_tol=0.0, seed=0) -> SthosvdResult:
    """`decide(mode, i, r, j) -> 0/1/2` is the Strategy hook (None = fixed EIG)."""
    x = _f(x)
    ranks = [int(r) for r in ranks]
    if len(ranks) != x.ndim:  # sthosvd.hpp:128-131
        from paper_2010_10131_b200.errors import RankExceedsDim

        raise RankExceedsDim(f"expected {x.ndim} truncations, got {len(ranks)}")
    box = {"err": None}

    def cb(_u, mode, i, r, j):
        try:
            return int(decide(int(mode), int(i), int(r), int(j))) if decide else 0
        except Exception as e:
            box["err"] = e
            return -1

    fn = SELECTOR_FN(cb)
    core = np.empty(ranks, order="F")
    factors = np.empty(sum(i * r for i, r in zip(x.shape, ranks)))
    reps = np.zeros((x.ndim, 5))
    code = load().or_sthosvd(_p(x), _d(x.shape), x.ndim, _d(ranks), fn, None, int(num_iters),
                             float(rel_tol), int(seed), _p(core), _p(factors), _p(reps))
    if box["err"] is not None:
        raise box["err"]
    _check(code)
    out, off = [], 0
    for i, r in zip(x.shape, ranks):
        out.append(np.asfortranarray(factors[off:off + i * r].reshape((i, r), order="F")))
        off += i * r
    return SthosvdResult(core, out, reps)


def _flat(factors) -> np.ndarray:
    return np.concatenate([_f(f).ravel(order="F") for f in factors])


def reconstruct(core, factors, original_dims) -> np.ndarray:
    core = _f(core)
    out = np.empty(original_dims, order="F")
    fl = _flat(factors)
    _check(load().or_reconstruct(_p(core), _d(core.shape), core.ndim, _p(fl), _d(original_dims), _p(out)))
    return out


def relative_error(x, core, factors) -> float:
    x, core = _f(x), _f(core)
    fl = _flat(factors)
    out = C.c_double()
    _check(load().or_relative_error(_p(x), _d(x.shape), x.ndim, _p(core), _d(core.shape), _p(fl),
                                    C.byref(out)))
    return out.value


def synth_lowrank(dims, ranks, seed: int) -> np.ndarray:
    out = np.empty(dims, order="F")
    _check(load().or_synth_lowrank(_d(dims), _d(ranks), len(dims), C.c_uint64(seed), _p(out)))
    return out


# ------------------------------------------------------------------ instrumentation / timers
def reset_counters() -> None:
    load().or_reset_counters()


def gemm_calls() -> int:
    return int(load().or_gemm_calls())


def gemm_flops() -> int:
    return int(load().or_gemm_flops())


def stage_times() -> dict:
    buf = (C.c_double * 4)()
    load().or_stage_times(buf)
    return {"gram_s": buf[0], "eig_s": buf[1], "ttm_s": buf[2], "als_s": buf[3]}


def cost_eig(i, r, j) -> float:
    return float(load().or_cost_eig(i, r, j))


def cost_als(i, r, j, iters=5) -> float:
    return float(load().or_cost_als(i, r, j, iters))


def __getattr__(name):  # pragma: no cover
    raise AttributeError(name)


os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")


def sthosvd_f32_eig0(x32, ranks, decide=None, threads=0, num_iters=5, rel_tol=0.0, seed=0) -> SthosvdResult:
    """Memory-lean oracle for big fp32 tensors (C5): mode 0 EIG streamed in fp64
    chunks, later modes through the regular restatement (see atk_oracle.cpp)."""
    x32 = np.asfortranarray(x32, dtype=np.float32)
    ranks = [int(r) for r in ranks]
    lib = load()
    lib.or_sthosvd_f32_eig0.argtypes = [C.POINTER(C.c_float), _up, C.c_int, _up, SELECTOR_FN, C.c_void_p, C.c_int,
                                        C.c_double, C.c_uint64, _dp, _dp, C.c_int]
    box = {"err": None}

    def cb(_u, mode, i, r, j):
        try:
            return int(decide(int(mode), int(i), int(r), int(j))) if decide else 0
        except Exception as e:
            box["err"] = e
            return -1

    fn = SELECTOR_FN(cb)
    core = np.empty(ranks, order="F")
    factors = np.empty(sum(i * r for i, r in zip(x32.shape, ranks)))
    code = lib.or_sthosvd_f32_eig0(x32.ctypes.data_as(C.POINTER(C.c_float)), _d(x32.shape), x32.ndim, _d(ranks),
                                   fn, None, int(num_iters), float(rel_tol), int(seed), _p(core), _p(factors),
                                   int(threads))
    if box["err"] is not None:
        raise box["err"]
    _check(code)
    out, off = [], 0
    for i, r in zip(x32.shape, ranks):
        out.append(np.asfortranarray(factors[off:off + i * r].reshape((i, r), order="F")))
        off += i * r
    return SthosvdResult(core, out, np.zeros((x32.ndim, 5)))


def norm2_f32(x32) -> float:
    lib = load()
    lib.or_norm2_f32.restype = C.c_double
    lib.or_norm2_f32.argtypes = [C.POINTER(C.c_float), C.c_uint64]
    x32 = np.asfortranarray(x32, dtype=np.float32)
    return float(lib.or_norm2_f32(x32.ctypes.data_as(C.POINTER(C.c_float)), x32.size))
