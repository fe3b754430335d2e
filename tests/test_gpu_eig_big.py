"""Exact dense eigensolver above n = 200 (trd_big.cu): linalg::sym_eig_top_r
(linalg.hpp:101-123) on any spectrum in bounded time.

The reference's Eigen SelfAdjointEigenSolver (linalg.hpp:108) returns every
eigenpair of any symmetric input; the engine's ChFSI needs a spectral gap, so
flat spectra, indefinite inputs and r > 112 go to the grid-wide Householder
tridiagonalisation + bisection + inverse iteration.  Checked against LAPACK
(numpy eigh):
* eigenvalues within 1e-12 of the largest |eigenvalue| (the reference's KAT
  tolerance class, test_linalg.cpp:72-95);
* the sign rule (linalg.hpp:34-50);
* eigenvectors through principal angles, per vector where it is separated by
  a relative gap > 1e-6, and as one subspace otherwise (<= 1e-9);
* orthonormality of the returned block (<= 1e-12);
* bit-identical results on repeated calls (the sharded path needs identical
  factors on every rank).
"""
import numpy as np
import pytest

from conftest import orthonormality_defect, principal_angle

pytestmark = pytest.mark.gpu


@pytest.fixture
def dctx():
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    yield ctx
    ctx.set_option("eig_method", -1)
    ctx.set_option("eig_assume_psd", 0.0)
    ctx.set_option("eig_dense_passes", 3)


def _check(s, r, res, vec_tol=1e-9):
    w, q = np.linalg.eigh(s)
    w, q = w[::-1], q[:, ::-1]
    scale = np.abs(w).max()
    assert np.abs(res.values - w[:r]).max() <= 1e-12 * scale, np.abs(res.values - w[:r]).max() / scale
    v = res.vectors
    assert orthonormality_defect(v) <= 1e-12
    for j in range(r):
        assert v[np.argmax(np.abs(v[:, j])), j] > 0
    # vectors: separated ones one by one, clusters as subspaces; the wanted block as a whole
    if r < len(w) and w[r - 1] - w[r] > 1e-6 * scale:
        assert principal_angle(v, q[:, :r]) <= vec_tol
    j = 0
    while j < r:
        e = j + 1
        while e < len(w) and w[e - 1] - w[e] <= 1e-6 * scale:
            e += 1
        if e <= r:
            assert principal_angle(v[:, j:e], q[:, j:e]) <= vec_tol, (j, e)
        j = e


def _sym(n, seed, kind):
    rng = np.random.default_rng(seed)
    if kind == "indefinite":
        a = rng.standard_normal((n, n))
        return 0.5 * (a + a.T)
    if kind == "flat_gram":  # Gram of uniform data: Marchenko-Pastur, no gap at r
        x = rng.uniform(-1, 1, (n, 3 * n))
        return x @ x.T
    if kind == "lowrank":
        q = np.linalg.qr(rng.standard_normal((n, n)))[0]
        lam = np.concatenate([np.linspace(4, 1, 64) * 1e4, rng.uniform(0.9, 1.1, n - 64)])
        return (q * lam) @ q.T
    if kind == "degenerate":  # repeated eigenvalues (clusters of 4)
        q = np.linalg.qr(rng.standard_normal((n, n)))[0]
        lam = np.repeat(np.linspace(10, 1, n // 4), 4)[:n]
        lam = np.concatenate([lam, np.ones(n - len(lam))])
        return (q * lam) @ q.T
    raise ValueError(kind)


@pytest.mark.parametrize("n,r,kind", [
    (201, 20, "indefinite"), (256, 64, "flat_gram"), (300, 1, "indefinite"), (517, 33, "lowrank"),
    (640, 150, "indefinite"), (1024, 32, "flat_gram"), (1024, 64, "degenerate"), (1500, 8, "flat_gram"),
])
def test_dense_big_matches_lapack(dctx, n, r, kind):
    from paper_2010_10131_b200 import atucker

    dctx.set_option("eig_method", 3)
    s = _sym(n, n + r, kind)
    _check(s, r, atucker.sym_eig_top_r(s, r, ctx=dctx))


def test_dense_big_2048_flat_deterministic(dctx):
    """C5's size on a flat Gram spectrum (uniform data): exact, and bit-identical twice."""
    from paper_2010_10131_b200 import atucker

    dctx.set_option("eig_method", 3)
    s = _sym(2048, 7, "flat_gram")
    a = atucker.sym_eig_top_r(s, 64, ctx=dctx)
    b = atucker.sym_eig_top_r(s, 64, ctx=dctx)
    assert np.array_equal(a.values, b.values) and np.array_equal(a.vectors, b.vectors)
    _check(s, 64, a)


def test_auto_flat_2048_falls_back_exact(dctx):
    """Default dispatch on a flat PSD Gram at n = 2048: ChFSI hands over to the
    dense solver after its pass budget; the result is exact either way."""
    from paper_2010_10131_b200 import atucker

    dctx.set_option("eig_assume_psd", 1.0)
    s = _sym(2048, 11, "flat_gram")
    _check(s, 64, atucker.sym_eig_top_r(s, 64, ctx=dctx))


def test_large_rank_above_chfsi_block(dctx):
    """r > 112 with n > 200 (previously ATK_UNSUPPORTED): the dense path takes it."""
    from paper_2010_10131_b200 import atucker

    s = _sym(400, 3, "indefinite")
    _check(s, 128, atucker.sym_eig_top_r(s, 128, ctx=dctx))


@pytest.mark.parametrize("n", [700, 1024, 1300])
def test_grid_only_reduction(dctx, n, monkeypatch):
    """The grid phase alone (no 16-CTA cluster tail): same exactness."""
    from paper_2010_10131_b200 import atucker

    monkeypatch.setenv("ATK_TRD_NOCLUSTER", "1")
    dctx.set_option("eig_method", 3)
    s = _sym(n, 5, "indefinite")
    _check(s, 24, atucker.sym_eig_top_r(s, 24, ctx=dctx))


def test_warp_backtransform_matches(dctx, monkeypatch):
    """The one-warp-per-vector back-transformation (kept for n where the blocked
    WY kernel's shared-memory block does not fit) on the same input."""
    from paper_2010_10131_b200 import atucker

    dctx.set_option("eig_method", 3)
    s = _sym(900, 13, "flat_gram")
    monkeypatch.setenv("ATK_BACKTR_WARP", "1")
    _check(s, 40, atucker.sym_eig_top_r(s, 40, ctx=dctx))


@pytest.mark.parametrize("n,r", [(2049, 10), (2156, 300), (3000, 64)])
def test_dense_above_2048(dctx, n, r):
    """2048 < n <= 4096 (kBigEigMax): the grid phase runs its <8, 32> instance, whose shared-memory
    layout beside the column slots is sized for 32 columns per CTA (an undersized layout wrote out
    of bounds for every n > 2048 before round 2's fix)."""
    from paper_2010_10131_b200 import atucker

    dctx.set_option("eig_method", 3)
    s = _sym(n, n, "indefinite")
    _check(s, r, atucker.sym_eig_top_r(s, r, ctx=dctx))
