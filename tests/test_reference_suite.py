"""The reference's own test suites, restated once and run on BOTH
implementations: `oracle` (CPU, pins the restatement) and `engine` (the
CUDA path through the C ABI, `-m gpu`).

Sources: proj/tests/test_kernels.cpp, test_linalg.cpp, test_solvers.cpp,
test_sthosvd.cpp, acceptance.cpp (cited per test).  Tolerances are the
reference's, made relative where the reference's absolute bound is
scale-dependent (test_output.txt:21 shows the reference failing its own 1e-12
absolute bound).
"""
import numpy as np
import pytest

import impls
from conftest import orthonormality_defect, principal_angle, random_signed
from paper_2010_10131_b200 import errors as E
from paper_2010_10131_b200.selector import (CostModelParams, DecisionTreeModel, Node, SolverKind,
                                            Strategy, cost_eig)

IMPLS = ["oracle", pytest.param("engine", marks=pytest.mark.gpu)]


@pytest.fixture(params=IMPLS)
def impl(request):
    return impls.get(request.param)


def uniform_signed(dims, seed):
    return random_signed(dims, seed, "uniform")


def random_matrix(rows, cols, seed, dist="uniform"):
    return random_signed([rows, cols], seed, dist)


def rng_dims(rng, order, lo, hi):
    return [int(v) for v in rng.integers(lo, hi + 1, size=order)]


# ---- independent index-walk oracles (oracles.hpp:29-87) -------------------------------
def unfold(x, n):
    return np.moveaxis(x, n, 0).reshape(x.shape[n], -1, order="F")


def ttm_explicit(x, u, n):
    y = np.tensordot(u, x, axes=([1], [n]))  # r x (other dims)
    return np.moveaxis(y, 0, n)


def ttt_explicit(x, y, n):
    return unfold(x, n) @ unfold(y, n).T


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(1e-300, np.abs(b).max()))


# ======================================================================= tensor
def test_frobenius_norm_basics(impl):
    """test_tensor.cpp:29-37 (tensor.hpp:158-168)."""
    assert impl.frobenius_norm(np.zeros((2, 2, 2), order="F")) == 0.0
    assert abs(impl.frobenius_norm(np.ones((2, 2, 2), order="F")) - np.sqrt(8.0)) <= 1e-12
    iota = np.arange(1.0, 9.0).reshape((2, 2, 2), order="F")  # sum of squares 204
    assert abs(impl.frobenius_norm(iota) - np.sqrt(204.0)) <= 1e-12


def test_frobenius_norm_matches_every_unfolding(impl):
    """test_tensor.cpp:39-51: the norm of every mode-n unfolding equals the tensor's."""
    rng = np.random.default_rng(11)
    for rep in range(20):
        order = 2 + rep % 3
        x = random_signed(rng_dims(rng, order, 2, 7), int(rng.integers(1 << 62)), "normal")
        ref = impl.frobenius_norm(x)
        assert abs(ref - np.sqrt((x * x).sum())) <= 1e-13 * ref
        for n in range(order):
            assert abs(impl.frobenius_norm(np.asfortranarray(unfold(x, n))) - ref) <= 1e-13 * ref


# ======================================================================= kernels
def test_ttm_identity_and_ones(impl):
    """test_kernels.cpp:34-49."""
    x = uniform_signed([3, 4, 5], 1)
    for n in range(3):
        y = impl.ttm(x, np.eye(x.shape[n]), n)
        assert np.abs(y - x).max() <= 1e-15
    ones = np.ones((2, 3, 4), order="F")
    y = impl.ttm(ones, np.ones((2, 3)), 1)
    assert y.shape == (2, 2, 4)
    assert np.all(y == 3.0)
    with pytest.raises(E.ShapeMismatch):
        impl.ttm(ones, np.ones((2, 3)), 0)
    with pytest.raises(E.ModeOutOfRange):
        impl.ttm(ones, np.ones((2, 3)), 3)


def test_ttm_matches_explicit(impl):
    """test_kernels.cpp:51-65 (50 random shapes, orders 2-4, r may exceed I_n)."""
    rng = np.random.default_rng(42)
    for rep in range(50):
        order = 2 + rep % 3
        x = uniform_signed(rng_dims(rng, order, 2, 9), int(rng.integers(1 << 62)))
        for n in range(order):
            r = 1 + int(rng.integers(0, x.shape[n] + 2))
            u = random_matrix(r, x.shape[n], int(rng.integers(1 << 62)))
            assert rel(impl.ttm(x, u, n), ttm_explicit(x, u, n)) <= 1e-12


def test_ttt_basics_and_explicit(impl):
    """test_kernels.cpp:67-95."""
    ones = np.ones((2, 3, 4), order="F")
    assert np.all(impl.ttt(ones, ones, 0) == 12.0)
    x = uniform_signed([4, 3, 5], 3)
    g = impl.ttt(x, x, 0)
    assert np.abs(g - g.T).max() <= 1e-13
    rng = np.random.default_rng(77)
    for rep in range(50):
        order = 2 + rep % 3
        dims = rng_dims(rng, order, 2, 8)
        a = uniform_signed(dims, int(rng.integers(1 << 62)))
        n = rep % order
        ydims = list(dims)
        ydims[n] = 1 + int(rng.integers(0, 6))
        b = uniform_signed(ydims, int(rng.integers(1 << 62)))
        assert rel(impl.ttt(a, b, n), ttt_explicit(a, b, n)) <= 1e-12
    with pytest.raises(E.ShapeMismatch):
        impl.ttt(x, uniform_signed([4, 3, 6], 5), 0)


def test_gram_is_symmetrized_self_ttt(impl):
    """test_kernels.cpp:97-114."""
    ones = np.ones((2, 3, 4), order="F")
    assert np.all(impl.gram(ones, 1) == 8.0)
    x = uniform_signed([4, 5, 6], 9)
    for n in range(3):
        g = impl.gram(x, n)
        assert rel(g, ttt_explicit(x, x, n)) <= 1e-12
        assert np.array_equal(g, g.T)  # exact symmetry
        vals, _ = impl.eig(g, g.shape[0])
        assert vals.min() >= -1e-10


def test_flop_charges(impl):
    """test_kernels.cpp:170-187 — I^2 J for gram, 2RIJ for ttm / ttt."""
    x = uniform_signed([4, 5, 6], 21)
    i, j = 5, 24
    impl.reset_counters()
    impl.gram(x, 1)
    assert impl.counters()[1] == i * i * j
    impl.reset_counters()
    impl.ttm(x, random_matrix(3, 5, 23), 1)
    assert impl.counters()[1] == 2 * 3 * i * j
    impl.reset_counters()
    impl.ttt(x, uniform_signed([4, 3, 6], 25), 1)
    assert impl.counters()[1] == 2 * i * 3 * j


def test_logical_gemm_counts(impl):
    """test_kernels.cpp:116-138.  The reference issues one Eigen GEMM per
    outer slab in the middle regime; the engine runs each contraction as ONE
    matricization-free kernel and records one logical GEMM per contraction."""
    rng = np.random.default_rng(123)
    for rep in range(10):
        order = 3 + rep % 2
        dims = rng_dims(rng, order, 2, 6)
        x = uniform_signed(dims, int(rng.integers(1 << 62)))
        for n in range(order):
            outer = int(np.prod(dims[n + 1:]))
            expected = 1 if (n == 0 or n + 1 == order or impl.name == "engine") else outer
            impl.reset_counters()
            impl.ttm(x, random_matrix(2, dims[n], 5), n)
            assert impl.counters()[0] == expected
            impl.reset_counters()
            impl.gram(x, n)
            assert impl.counters()[0] == expected


def test_ttm_norm_bound(impl):
    """test_kernels.cpp:158-168."""
    rng = np.random.default_rng(17)
    for rep in range(10):
        x = uniform_signed(rng_dims(rng, 3, 2, 7), int(rng.integers(1 << 62)))
        n = rep % 3
        u = random_matrix(1 + int(rng.integers(0, 5)), x.shape[n], int(rng.integers(1 << 62)))
        smax = np.linalg.svd(u, compute_uv=False)[0]
        assert np.linalg.norm(impl.ttm(x, u, n)) <= smax * np.linalg.norm(x) + 1e-10


# ======================================================================= linalg
def test_sym_eig_closed_forms(impl):
    """test_linalg.cpp:72-95."""
    d = np.diag([3.0, 1.0, 2.0])
    vals, vecs = impl.eig(d, 2)
    assert vals == pytest.approx([3.0, 2.0], abs=1e-12)
    assert vecs[0, 0] == pytest.approx(1.0, abs=1e-12)
    assert vecs[2, 1] == pytest.approx(1.0, abs=1e-12)
    s = np.array([[2.0, 1.0], [1.0, 2.0]])
    vals, vecs = impl.eig(s, 2)
    assert vals == pytest.approx([3.0, 1.0], abs=1e-12)
    h = 1 / np.sqrt(2)
    assert vecs[0, 0] == pytest.approx(h, abs=1e-12) and vecs[1, 0] == pytest.approx(h, abs=1e-12)
    assert abs(vecs[0, 1]) == pytest.approx(h, abs=1e-12)
    assert vecs[0, 1] + vecs[1, 1] == pytest.approx(0.0, abs=1e-12)
    with pytest.raises(E.NotSquare):
        impl.eig(random_matrix(2, 3, 5), 1)
    with pytest.raises(E.RankTooLarge):
        impl.eig(s, 3)


def test_sym_eig_full_spd_spectrum(impl):
    """test_linalg.cpp:97-109."""
    b = random_matrix(10, 8, 3, "normal")
    s = b.T @ b + 0.5 * np.eye(8)
    vals, vecs = impl.eig(s, 8)
    assert orthonormality_defect(vecs) <= 1e-10
    assert np.all(np.diff(vals) <= 0)
    assert np.abs((vecs * vals) @ vecs.T - s).max() <= 1e-10


def test_sign_rule(impl):
    """linalg.hpp:34-50 — largest-|v| entry of every vector is positive."""
    b = random_matrix(20, 12, 8, "normal")
    _, vecs = impl.eig(b.T @ b, 5)
    for j in range(5):
        k = int(np.argmax(np.abs(vecs[:, j])))
        assert vecs[k, j] > 0


def test_thin_qr_contracts(impl):
    """test_linalg.cpp:111-147."""
    q, r = impl.qr(np.eye(4))
    assert np.abs(q - np.eye(4)).max() <= 1e-14 and np.abs(r - np.eye(4)).max() <= 1e-14
    q, r = impl.qr(np.array([[3.0], [4.0]]))
    assert q[0, 0] == pytest.approx(0.6, abs=1e-14) and q[1, 0] == pytest.approx(0.8, abs=1e-14)
    assert r[0, 0] == pytest.approx(5.0, abs=1e-14)
    a = random_matrix(10, 4, 7, "normal")
    q, r = impl.qr(a)
    assert orthonormality_defect(q) <= 1e-12
    assert np.all(np.diag(r) >= 0) and np.all(np.tril(r, -1) == 0)
    assert np.linalg.norm(q @ r - a) / np.linalg.norm(a) <= 1e-13
    dfc = np.stack([np.arange(1, 6.0), 2 * np.arange(1, 6.0)], axis=1)
    with pytest.raises(E.RankDeficient):
        impl.qr(dfc)


def test_spd_solve_contracts(impl):
    """test_linalg.cpp:189-219."""
    b = random_matrix(4, 2, 17, "normal")
    assert np.abs(impl.spd_solve(np.eye(4), b) - b).max() <= 1e-14
    x = impl.spd_solve(np.diag([2.0, 4.0]), np.array([[2.0], [8.0]]))
    assert x[:, 0] == pytest.approx([1.0, 2.0], abs=1e-13)
    m = random_matrix(8, 6, 19, "normal")
    a = m.T @ m + 0.5 * np.eye(6)
    rb = random_matrix(6, 2, 23, "normal")
    sol = impl.spd_solve(a, rb)
    assert np.linalg.norm(a @ sol - rb) <= 1e-10 * np.linalg.norm(rb)
    with pytest.raises(E.NotSPD):
        impl.spd_solve(np.diag([1.0, -1.0]), np.array([[2.0], [8.0]]))


def test_eig_of_yyt_is_sigma_squared(impl):
    """test_linalg.cpp:221-228."""
    y = random_matrix(5, 12, 31, "normal")
    vals, _ = impl.eig(y @ y.T, 5)
    sig = np.linalg.svd(y, compute_uv=False)
    assert vals == pytest.approx(sig**2, rel=1e-9)


# ======================================================================= solvers
def test_eig_mode_exact_rank(impl, oracle):
    """test_solvers.cpp:43-50."""
    y = oracle.synth_lowrank([12, 10, 8], [3, 3, 3], 101)
    f, s = impl.eig_mode(y, 0, 3)
    assert abs(np.linalg.norm(y) - np.linalg.norm(s)) <= 1e-8 * np.linalg.norm(y)
    assert orthonormality_defect(f) <= 1e-10
    assert s.shape == (3, 10, 8)


def test_eig_mode_energy_identity(impl):
    """test_solvers.cpp:52-65."""
    y = random_signed([9, 8, 7], 5)
    for n in range(3):
        vals, _ = impl.eig(impl.gram(y, n), y.shape[n])
        _, s = impl.eig_mode(y, n, 4)
        assert np.linalg.norm(s) ** 2 == pytest.approx(vals[:4].sum(), rel=1e-8)


def test_eig_mode_full_rank_and_subspace(impl):
    """test_solvers.cpp:67-85."""
    y = random_signed([6, 5, 4], 7)
    f, s = impl.eig_mode(y, 1, 5)
    back = ttm_explicit(s, f, 1)
    assert np.abs(back - y).max() / np.linalg.norm(y) <= 1e-10
    y = random_signed([6, 5, 4], 9)
    for n in range(3):
        u, sig, _ = np.linalg.svd(unfold(y, n), full_matrices=False)
        if sig[1] - sig[2] <= 1e-6:
            continue
        f, _ = impl.eig_mode(y, n, 2)
        assert principal_angle(f, u[:, :2]) <= 1e-6


def _fit(y, l, rfac, n):
    return np.linalg.norm(unfold(y, n) - l @ unfold(rfac, n))


def test_als_iterate_contracts(impl, oracle):
    """test_solvers.cpp:87-144."""
    y = oracle.synth_lowrank([10, 9, 8], [3, 3, 3], 11)
    l0 = oracle.random_tensor([10, 3], 13, "normal")
    l, rfac, it = impl.als_iterate(y, 0, l0)
    assert it == 5
    assert _fit(y, l, rfac, 0) <= 1e-6 * np.linalg.norm(y)
    z = random_signed([5, 6, 4], 17)
    l, rfac, _ = impl.als_iterate(z, 0, np.eye(5), num_iters=1)
    assert _fit(z, l, rfac, 0) <= 1e-12 * np.linalg.norm(z)
    # monotone objective: replay k = 1..5 iterations from the same start
    w = random_signed([8, 7, 6], 19)
    l0 = oracle.random_tensor([7, 3], 23, "normal")
    obj = [_fit(w, *impl.als_iterate(w, 1, l0, num_iters=k)[:2], 1) for k in range(1, 6)]
    assert all(obj[k] <= obj[k - 1] + 1e-9 for k in range(1, 5))
    # degenerate start -> NotSPD
    bad = np.zeros((5, 2))
    bad[:, 0] = 1.0
    with pytest.raises(E.NotSPD):
        impl.als_iterate(random_signed([5, 4, 3], 29), 0, bad)
    # rel_tol early stop
    ylr = oracle.synth_lowrank([10, 8, 6], [2, 2, 2], 31)
    _, _, it = impl.als_iterate(ylr, 0, oracle.random_tensor([10, 2], 37, "normal"), num_iters=50,
                                rel_tol=1e-12)
    assert it < 50


def test_als_mode_solver(impl, oracle):
    """test_solvers.cpp:146-159."""
    y = oracle.synth_lowrank([12, 10, 8], [3, 3, 3], 41)
    f, s, _ = impl.als_mode(y, 0, 3, seed=1)
    assert orthonormality_defect(f) <= 1e-10
    assert np.abs(ttm_explicit(s, f, 0) - y).max() / np.linalg.norm(y) <= 1e-6
    z = random_signed([6, 5, 4], 43)
    f, s, _ = impl.als_mode(z, 1, 5, seed=1)
    assert np.abs(ttm_explicit(s, f, 1) - z).max() / np.linalg.norm(z) <= 1e-10
    assert s.shape == (6, 5, 4)


def test_svd_mode_solver(impl):
    """test_solvers.cpp:177-201."""
    d = np.zeros((3, 3, 1), order="F")
    d[0, 0, 0], d[1, 1, 0], d[2, 2, 0] = 5.0, 3.0, 1.0
    f, _ = impl.svd_mode(d, 0, 2)
    assert abs(f[0, 0]) == pytest.approx(1.0, abs=1e-12)
    assert abs(f[1, 1]) == pytest.approx(1.0, abs=1e-12)
    assert f[1, 0] == pytest.approx(0.0, abs=1e-12)
    y = random_signed([6, 5, 4], 53)
    f, s = impl.svd_mode(y, 2, 4)
    assert np.abs(ttm_explicit(s, f, 2) - y).max() / np.linalg.norm(y) <= 1e-12
    y = random_signed([6, 5, 4], 59)
    for n in range(3):
        _, se = impl.eig_mode(y, n, 3)
        _, ss = impl.svd_mode(y, n, 3)
        assert np.linalg.norm(se) == pytest.approx(np.linalg.norm(ss), rel=1e-9)


def test_solver_preconditions(impl):
    """test_solvers.cpp:203-209."""
    y = random_signed([4, 3, 2], 61)
    with pytest.raises(E.RankExceedsDim):
        impl.eig_mode(y, 0, 5)
    with pytest.raises(E.RankExceedsDim):
        impl.eig_mode(y, 0, 0)
    with pytest.raises(E.RankExceedsDim):
        impl.als_mode(y, 1, 4)
    with pytest.raises(E.ModeOutOfRange):
        impl.svd_mode(y, 3, 1)


def test_shrunk_dims_every_solver(impl):
    """test_solvers.cpp:211-228."""
    y = random_signed([7, 6, 5, 4], 67)
    for n in range(4):
        outs = [impl.eig_mode(y, n, 2), impl.als_mode(y, n, 2)[:2], impl.svd_mode(y, n, 2)]
        for f, s in outs:
            want = list(y.shape)
            want[n] = 2
            assert list(s.shape) == want and f.shape == (y.shape[n], 2)
            assert orthonormality_defect(f) <= 1e-10


# ======================================================================= driver
def test_exact_rank_every_strategy(impl, oracle):
    """test_sthosvd.cpp:39-52."""
    x = oracle.synth_lowrank([20, 30, 40], [5, 6, 7], 2024)
    for s in [Strategy.fixed_eig(), Strategy.fixed_als(), Strategy.fixed_svd(), Strategy.cost_model()]:
        core, factors, _ = impl.sthosvd(x, [5, 6, 7], s, seed=3)
        assert impl.relative_error(x, core, factors) <= 1e-8
        assert core.shape == (5, 6, 7)


def test_full_rank_and_eig_vs_svd(impl):
    """test_sthosvd.cpp:54-68."""
    x = random_signed([8, 7, 6], 5)
    core, f, _ = impl.sthosvd(x, [8, 7, 6])
    assert impl.relative_error(x, core, f) <= 1e-12
    for seed in (1, 2, 3):
        x = random_signed([12, 10, 8], seed)
        ce, fe, _ = impl.sthosvd(x, [4, 3, 2], Strategy.fixed_eig())
        cs, fs, _ = impl.sthosvd(x, [4, 3, 2], Strategy.fixed_svd())
        assert abs(impl.relative_error(x, ce, fe) - impl.relative_error(x, cs, fs)) <= 1e-10


def test_reconstruct_kats(impl):
    """test_sthosvd.cpp:70-95."""
    x = random_signed([4, 3, 2], 7)
    y = impl.reconstruct(x, [np.eye(4), np.eye(3), np.eye(2)], [4, 3, 2])
    assert np.abs(y - x).max() == 0.0
    u = np.array([[0.5], [-0.5], [0.5], [-0.5]])
    v = np.array([[1 / np.sqrt(2)], [0.0], [-1 / np.sqrt(2)]])
    w = np.array([[0.6], [0.8]])
    full = impl.reconstruct(np.full((1, 1, 1), 2.5), [u, v, w], [4, 3, 2])
    want = 2.5 * np.einsum("i,j,k->ijk", u[:, 0], v[:, 0], w[:, 0])
    assert np.abs(full - want).max() <= 1e-14


def test_relative_error_special_cases(impl):
    """test_sthosvd.cpp:97-108."""
    x = random_signed([5, 4, 3], 11)
    core, f, _ = impl.sthosvd(x, [5, 4, 3])
    assert impl.relative_error(x, core, f) <= 1e-12
    assert impl.relative_error(x, np.zeros_like(core), f) == pytest.approx(1.0, abs=1e-12)
    with pytest.raises(E.ZeroNormInput):
        impl.relative_error(np.zeros((2, 2)), np.zeros((2, 2)), [np.eye(2), np.eye(2)])


def test_reports_chain_and_adaptive_hook(impl):
    """test_sthosvd.cpp:110-151 — decisions recorded, hook sees the shrunk J."""
    x = random_signed([9, 8, 7], 13)
    _, _, used = impl.sthosvd(x, [3, 4, 5], Strategy.manual([SolverKind.Eig, SolverKind.Als,
                                                              SolverKind.Eig]))
    assert used == [0, 1, 0]
    seen = []

    class Spy(Strategy):
        def decide(self, mode, i, r, j, params=None):
            seen.append((mode, i, r, j))
            return SolverKind.Als

    model = DecisionTreeModel(nodes=[Node(leaf=True, label=1)], root=0)
    x = random_signed([6, 5, 4], 17)
    _, _, used = impl.sthosvd(x, [2, 2, 2], Strategy.adaptive(model))
    assert used == [1, 1, 1]
    impl.sthosvd(x, [2, 2, 2], Spy(Strategy.Kind.Adaptive, model=model))
    assert seen[1] == (1, 5, 2, 2 * 4)  # mode 0 already shrunk to 2
    assert cost_eig(5.0, 2.0, 8.0) == pytest.approx(cost_eig(5, 2, 8))


def test_manual_strategies_agree(impl):
    """test_sthosvd.cpp:153-169 (5 reps instead of 20)."""
    rng = np.random.default_rng(19)
    for rep in range(5):
        x = random_signed(rng_dims(rng, 3, 24, 34), int(rng.integers(1 << 62)))
        ranks = [max(2, d // 3) for d in x.shape]
        errs = []
        for mask in range(8):
            s = Strategy.manual([SolverKind.Als if (mask >> n) & 1 else SolverKind.Eig for n in range(3)])
            core, f, _ = impl.sthosvd(x, ranks, s, seed=23)
            errs.append(impl.relative_error(x, core, f))
        assert max(errs) - min(errs) <= 0.01


def test_core_energy_accounting(impl):
    """test_sthosvd.cpp:171-188."""
    x = random_signed([10, 9, 8], 29)
    work, discarded = x, 0.0
    for n, r in enumerate([4, 4, 4]):
        vals, _ = impl.eig(impl.gram(work, n), work.shape[n])
        discarded += vals[r:].sum()
        _, work = impl.eig_mode(work, n, r)
    assert np.linalg.norm(work) ** 2 + discarded == pytest.approx(np.linalg.norm(x) ** 2, rel=1e-6)


def test_driver_validation_and_error_context(impl):
    """test_sthosvd.cpp:190-205."""
    x = random_signed([5, 4, 3], 31)
    with pytest.raises(E.RankExceedsDim):
        impl.sthosvd(x, [5, 4])
    with pytest.raises(E.RankExceedsDim):
        impl.sthosvd(x, [5, 4, 9])
    with pytest.raises(E.Error):
        impl.sthosvd(x, [1, 1, 1], Strategy.manual([SolverKind.Eig]))
    with pytest.raises(E.Error):
        Strategy.manual([SolverKind.Svd])
    thin = random_signed([9, 2, 2], 37)
    with pytest.raises(E.Error, match="mode 1"):
        impl.sthosvd(thin, [5, 1, 1], Strategy.fixed_svd())


# ======================================================================= acceptance.cpp
def test_acceptance_kernel_equivalence(impl):
    """acceptance.cpp:65-99 criterion 1 (relative form; 40 tensors, dims <= 20)."""
    rng = np.random.default_rng(1)
    worst = 0.0
    for rep in range(40):
        order = 3 + rep % 2
        x = random_signed(rng_dims(rng, order, 2, 20 if order == 3 else 8), int(rng.integers(1 << 62)))
        n = rep % order
        worst = max(worst, rel(impl.gram(x, n), ttt_explicit(x, x, n)))
        u = random_matrix(3, x.shape[n], 9, "normal")
        worst = max(worst, rel(impl.ttm(x, u, n), ttm_explicit(x, u, n)))
    assert worst <= 1e-12


def test_acceptance_eig_als_svd_agreement(impl):
    """acceptance.cpp:179-197 criterion 5 (5 tensors of 30^3, r = 10)."""
    for seed in range(5):
        x = random_signed([30, 30, 30], 1000 + seed)
        ce, fe, _ = impl.sthosvd(x, [10, 10, 10], Strategy.fixed_eig())
        ca, fa, _ = impl.sthosvd(x, [10, 10, 10], Strategy.fixed_als(), seed=seed)
        cs, fs, _ = impl.sthosvd(x, [10, 10, 10], Strategy.fixed_svd())
        ee = impl.relative_error(x, ce, fe)
        assert abs(ee - impl.relative_error(x, ca, fa)) <= 0.01
        assert abs(ee - impl.relative_error(x, cs, fs)) <= 1e-9
