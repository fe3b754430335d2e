"""svd_mode_solver on the explicit unfolding (csrc/svd.cu) against the
reference's thin SVD (solvers.hpp:142-162, linalg.hpp:153-166; the oracle runs
LAPACK dgesdd on the same matricized Y).

The unfolding is built as U diag(sigma) V^T with sigma spread over 1 .. 1e-10,
so the Gram route (sigma = sqrt(lambda of Y Y^T)) cannot resolve the left
singular vectors below sigma_k / sigma_1 ~ 1e-8 (their eigenvalues sit under
eps * lambda_1): the explicit route must match the truth (and dgesdd) there,
the Gram route must not (the test has teeth).  Tolerances: per-vector
principal angle <= 1e-5 (dgesdd's own error for sigma_k = 1e-10 sigma_1 at a
relative gap of ~0.4 is ~eps / (1e-10 * 0.4) ~ 6e-6), sigma relative <= 1e-5.
"""
import numpy as np
import pytest

from conftest import principal_angle

pytestmark = pytest.mark.gpu


def _graded(dims, mode, sig, seed):
    rng = np.random.default_rng(seed)
    i = dims[mode]
    j = int(np.prod(dims)) // i
    k = len(sig)
    u = np.linalg.qr(rng.standard_normal((i, k)))[0]
    v = np.linalg.qr(rng.standard_normal((j, k)))[0]
    m = (u * sig) @ v.T  # the mode-n unfolding, I x J
    rest = [d for q, d in enumerate(dims) if q != mode]
    y = np.moveaxis(m.reshape([i] + rest, order="F"), 0, mode)
    return np.asfortranarray(y), u


@pytest.fixture
def sctx():
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    yield ctx
    ctx.set_option("svd_explicit", 1)


@pytest.mark.parametrize("dims,mode,r", [([40, 30, 20], 0, 30), ([24, 40, 25], 1, 30), ([16, 12, 60], 2, 50),
                                         # tall unfoldings (I > J): the column-rotated mirror path
                                         ([60, 4, 5], 0, 15), ([3, 90, 8], 1, 20), ([4, 5, 300], 2, 20)])
def test_svd_mode_ill_conditioned(sctx, oracle, dims, mode, r):
    from paper_2010_10131_b200 import atucker

    k = min(dims[mode], int(np.prod(dims)) // dims[mode])
    sig = np.logspace(0, -10, k)
    y, u_true = _graded(dims, mode, sig, 7 + mode)
    res = atucker.svd_mode_solver(y, mode, r, ctx=sctx)
    ref = oracle.svd_mode_solver(y, mode, r)
    u = res.factor
    # per vector against the truth and against dgesdd (sign rule: identical columns)
    ang = [principal_angle(u[:, [q]], u_true[:, [q]]) for q in range(r)]
    assert max(ang) <= 1e-5, max(ang)
    assert np.abs(u - ref.factor).max() <= 1e-5
    # shrunk rows = sigma_k v_k^T: norms are the singular values, relative to each
    sh = np.moveaxis(np.asarray(res.shrunk), mode, 0).reshape(r, -1, order="F")
    sref = np.moveaxis(ref.shrunk, mode, 0).reshape(r, -1, order="F")
    s_got = np.linalg.norm(sh, axis=1)
    assert np.all(np.abs(s_got - sig[:r]) <= 1e-5 * sig[:r])
    assert np.all(np.abs(sh - sref).max(axis=1) <= 1e-5 * sig[:r] + 1e-14)
    # the Gram route loses the small-sigma vectors
    sctx.set_option("svd_explicit", 0)
    g = atucker.svd_mode_solver(y, mode, r, ctx=sctx).factor
    assert max(principal_angle(g[:, [q]], u_true[:, [q]]) for q in range(r)) > 1e-3


def test_svd_mode_matches_oracle_well_conditioned(sctx, oracle):
    """A plain random fp64 tensor: factor and shrunk equal dgesdd's to 1e-10."""
    from paper_2010_10131_b200 import atucker

    y = np.asfortranarray(np.random.default_rng(3).standard_normal((30, 20, 25)))
    for mode, r in [(0, 10), (1, 20), (2, 5)]:
        res = atucker.svd_mode_solver(y, mode, r, ctx=sctx)
        ref = oracle.svd_mode_solver(y, mode, r)
        assert np.abs(res.factor - ref.factor).max() <= 1e-10
        assert np.abs(np.asarray(res.shrunk) - ref.shrunk).max() <= 1e-10 * np.abs(ref.shrunk).max()


def test_sthosvd_fixed_svd_explicit(sctx, oracle):
    """sthosvd with Strategy::fixed_svd (every mode on the explicit route) vs the oracle."""
    from paper_2010_10131_b200 import atucker
    from paper_2010_10131_b200.selector import Strategy

    x = np.asfortranarray(np.random.default_rng(5).standard_normal((24, 18, 20)))
    res = atucker.sthosvd(x, [6, 5, 4], Strategy.fixed_svd(), ctx=sctx)
    ref = oracle.sthosvd(x, [6, 5, 4], lambda m, i, r, j: 2)
    assert abs(np.linalg.norm(res.decomposition.core) - np.linalg.norm(ref.core)) <= 1e-10 * np.linalg.norm(ref.core)
    for a, b in zip(res.decomposition.factors, ref.factors):
        assert np.abs(a - b).max() <= 1e-9
    assert all(rp.eig_method == "svd-jacobi" for rp in res.reports)


def test_svd_mode_tall_rank_deficient_matches_oracle(sctx, oracle):
    """test_sthosvd.cpp:39-52 on the SVD route: the last mode of a [20, 30, 40] exact-rank
    tensor shrunk to 5 x 6 is a 40 x 30 unfolding of rank 7 (I > J)."""
    from paper_2010_10131_b200 import atucker
    from paper_2010_10131_b200.selector import Strategy

    x = oracle.synth_lowrank([20, 30, 40], [5, 6, 7], 2024)
    res = atucker.sthosvd(x, [5, 6, 7], Strategy.fixed_svd(), ctx=sctx)
    ref = oracle.sthosvd(x, [5, 6, 7], lambda m, i, r, j: 2)
    assert atucker.relative_error(x, res.decomposition, ctx=sctx) <= 1e-8
    for a, b in zip(res.decomposition.factors, ref.factors):
        assert principal_angle(a, b) <= 1e-8


@pytest.mark.parametrize("rank", [0, 1, 4])
def test_svd_mode_tall_rank_below_r_completes_basis(sctx, oracle, rank):
    """A 40 x 12 (tall) unfolding of rank < r = 8: the columns whose sigma is at rounding level carry
    no direction and are completed to an orthonormal basis (Eigen's JacobiSVD U is orthonormal for
    zero singular values too, linalg.hpp:153-166); the rank-`rank` part matches the oracle."""
    from paper_2010_10131_b200 import atucker

    rng = np.random.default_rng(40 + rank)
    y = np.asfortranarray(rng.standard_normal((40, rank)) @ rng.standard_normal((rank, 12)))
    res = atucker.svd_mode_solver(y, 0, 8, ctx=sctx)
    u = np.asarray(res.factor)
    assert np.abs(u.T @ u - np.eye(8)).max() <= 1e-12
    assert np.linalg.norm(y - u @ (u.T @ y)) <= 1e-12 * max(np.linalg.norm(y), 1e-300)
    if rank:
        ref = oracle.svd_mode_solver(y, 0, 8)
        assert principal_angle(u[:, :rank], np.asarray(ref.factor)[:, :rank]) <= 1e-10
