"""Device symmetric eigensolver (linalg::sym_eig_top_r, linalg.hpp:101-123).

The default dense solver (tridiag.cu: Householder + bisection + inverse
iteration, n <= 200) is covered by tests/test_gpu_tridiag.py and by the
"auto" parametrisation here.  Both Jacobi variants of jacobi.cu are checked against LAPACK (numpy eigh):
* the general one (indefinite input: the API default);
* the Cholesky-preconditioned, vector-free PSD one ("eig_assume_psd"). This
  includes rank-deficient Grams, where the shift keeps the factorisation
  definite, and an indefinite input, which must fall back to the general
  variant.
ChFSI (n > 112) is covered on gapped and flat PSD spectra.

Tolerances: eigenvalues 1e-12 relative to the largest. Eigenvectors are compared
through the principal angle of each well-separated eigenvector (≤ 1e-9).
"""
import numpy as np
import pytest

from conftest import principal_angle

pytestmark = pytest.mark.gpu


def _check(s, r, res, vec_tol=1e-9):
    w, q = np.linalg.eigh(s)
    w, q = w[::-1][:r], q[:, ::-1][:, :r]
    scale = np.abs(np.linalg.eigvalsh(s)).max()
    assert np.abs(res.values - w).max() <= 1e-12 * scale
    # sign rule (linalg.hpp:34-50): largest-|.| entry of each column positive
    for j in range(r):
        v = res.vectors[:, j]
        assert v[np.argmax(np.abs(v))] > 0
    # vectors: only where the eigenvalue is separated from its neighbours
    full = np.linalg.eigvalsh(s)[::-1]
    for j in range(r):
        gap = min(abs(full[j] - full[j - 1]) if j > 0 else np.inf, abs(full[j] - full[j + 1]))
        if gap > 1e-6 * scale:
            assert principal_angle(res.vectors[:, j:j + 1], q[:, j:j + 1]) <= vec_tol


@pytest.fixture(params=[(False, 0), (True, 0), (False, -1)], ids=["jacobi-general", "jacobi-psd", "auto"])
def ectx(request):
    """Jacobi (eig_method 0, both variants) and the default dispatch (the
    tridiagonal solver for n <= 200, ChFSI above with tridiagonal Rayleigh-Ritz)."""
    from paper_2010_10131_b200 import atucker

    psd, method = request.param
    ctx = atucker.Context.default(0)
    ctx.set_option("eig_assume_psd", 1.0 if psd else 0.0)
    ctx.set_option("eig_method", method)
    yield ctx
    ctx.set_option("eig_assume_psd", 0.0)
    ctx.set_option("eig_method", -1)


@pytest.mark.parametrize("n", [2, 5, 17, 48, 96, 112, 128, 152])
def test_dense_gram(ectx, n):
    from paper_2010_10131_b200 import atucker

    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, n + 7))
    s = a @ a.T
    _check(s, max(1, n // 2), atucker.sym_eig_top_r(s, max(1, n // 2), ctx=ectx))


@pytest.mark.parametrize("n", [48, 96])
def test_dense_gapped_rr_block(ectx, n):
    """Rayleigh-Ritz-like block: 2/3 of the spectrum at 1e6 scale, the rest ~1."""
    from paper_2010_10131_b200 import atucker

    rng = np.random.default_rng(7)
    q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    top = 2 * n // 3
    lam = np.concatenate([rng.uniform(1, 4, top) * 1e6, rng.uniform(0.9, 1.1, n - top)])
    s = (q * lam) @ q.T
    _check(s, top, atucker.sym_eig_top_r(s, top, ctx=ectx))


def test_dense_rank_deficient_gram(ectx):
    from paper_2010_10131_b200 import atucker

    rng = np.random.default_rng(3)
    a = rng.standard_normal((80, 20))
    s = a @ a.T  # rank 20
    _check(s, 10, atucker.sym_eig_top_r(s, 10, ctx=ectx))


def test_dense_indefinite(ectx):
    """Indefinite input: with eig_assume_psd the Cholesky fails and the kernel
    falls back to the general variant; results must be identical in quality."""
    from paper_2010_10131_b200 import atucker

    rng = np.random.default_rng(11)
    b = rng.standard_normal((64, 64))
    s = (b + b.T) / 2
    _check(s, 12, atucker.sym_eig_top_r(s, 12, ctx=ectx))


@pytest.mark.parametrize("kind", ["gapped", "flat"])
@pytest.mark.parametrize("fused", [1, 0], ids=["cheb-fused", "cheb-steps"])
def test_chfsi(ectx, kind, fused):
    """ChFSI with the Chebyshev filter as one cooperative launch per pass
    (default) and as per-step launches; both must give the same quality."""
    from paper_2010_10131_b200 import atucker

    ectx.set_option("cheb_fused", fused)

    n, r = 640, 32
    rng = np.random.default_rng(5)
    q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    if kind == "gapped":
        lam = np.concatenate([np.sort(rng.uniform(1, 4, r))[::-1] * 1e6, rng.uniform(0.9, 1.1, n - r)])
    else:
        lam = np.sort(1.0 + 0.3 * rng.random(n))[::-1]
    s = (q * lam) @ q.T
    s = (s + s.T) / 2
    res = atucker.sym_eig_top_r(s, r, ctx=ectx)
    ectx.set_option("cheb_fused", 1)
    _check(s, r, res, vec_tol=1e-8 if kind == "gapped" else 1e-5)


@pytest.mark.parametrize("fused", [1, 2, 0], ids=["cheb-resident", "cheb-splitk", "cheb-steps"])
def test_chfsi_dominant_top(fused):
    """Gram of non-centred data: the mean direction's eigenvalue is ~1e3 x the
    rest.  Converged top pairs are locked and the filter runs on a deflated S
    (eig.cu); without locking the wanted-set dynamic-range cap would hold the
    filter at degree ~2 for ~100 passes.  Also compares the three Chebyshev
    filter implementations (resident-S clusters, split-K cooperative, per-step)."""
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    ctx.set_option("eig_assume_psd", 1.0)
    ctx.set_option("cheb_fused", fused)
    try:
        n, r = 512, 24
        rng = np.random.default_rng(9)
        a = rng.random((n, 3 * n))
        s = a @ a.T
        _check(s, r, atucker.sym_eig_top_r(s, r, ctx=ctx), vec_tol=1e-6)
    finally:
        ctx.set_option("cheb_fused", 1)
        ctx.set_option("eig_assume_psd", 0.0)


@pytest.mark.parametrize("tiles", [1, 0], ids=["lanczos-tiles", "lanczos-l2"])
def test_chfsi_indefinite_lanczos(tiles):
    """Indefinite input above the tridiagonal limit: the filter's lower bound
    comes from the Lanczos run, with S resident in a 16-CTA cluster or
    re-read from L2; both must converge to LAPACK's values."""
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    ctx.set_option("lanczos_tiles", tiles)
    try:
        n, r = 400, 20
        rng = np.random.default_rng(11)
        q = np.linalg.qr(rng.standard_normal((n, n)))[0]
        lam = np.concatenate([np.linspace(10.0, 6.0, r), rng.uniform(-4.0, 5.0, n - r)])
        s = (q * lam) @ q.T
        s = (s + s.T) / 2
        _check(s, r, atucker.sym_eig_top_r(s, r, ctx=ctx), vec_tol=1e-6)
    finally:
        ctx.set_option("lanczos_tiles", 1)


def test_chfsi_cheb_dataflow():
    """The resident Chebyshev filter with per-CTA ready flags instead of the grid
    barrier (option cheb_dataflow) on a flat spectrum: same bars as the default."""
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    ctx.set_option("eig_assume_psd", 1.0)
    ctx.set_option("cheb_dataflow", 1)
    try:
        n, r = 640, 32
        rng = np.random.default_rng(5)
        q = np.linalg.qr(rng.standard_normal((n, n)))[0]
        lam = np.sort(1.0 + 0.3 * rng.random(n))[::-1]
        s = (q * lam) @ q.T
        s = (s + s.T) / 2
        _check(s, r, atucker.sym_eig_top_r(s, r, ctx=ctx), vec_tol=1e-5)
    finally:
        ctx.set_option("cheb_dataflow", 0)
        ctx.set_option("eig_assume_psd", 0.0)


def test_chfsi_scratch_growth_and_stream_switch():
    """ChFSI's block buffers live in the context's persistent scratch: a larger block grows it, a
    smaller one reuses it, and switching the context's stream orders the reuse (the previous stream
    is synchronised).  Every solve must match numpy, and a result must not change when a later
    solve reuses the scratch."""
    import torch

    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context(0)
    rng = np.random.default_rng(11)

    def gapped(n, r):
        q = np.linalg.qr(rng.standard_normal((n, n)))[0]
        lam = np.concatenate([np.sort(rng.uniform(1, 4, r))[::-1] * 1e5, rng.uniform(0.9, 1.1, n - r)])
        s = (q * lam) @ q.T
        return (s + s.T) / 2

    cases = [(gapped(300, 8), 8), (gapped(700, 48), 48), (gapped(260, 12), 12)]
    side = torch.cuda.Stream()
    results = []
    for i, (s, r) in enumerate(cases):
        if i == 2:
            ctx.set_stream(side.cuda_stream)
        res = atucker.sym_eig_top_r(s, r, ctx=ctx)
        _check(s, r, res, vec_tol=1e-8)
        results.append(res)
    ctx.set_stream(0)
    again = atucker.sym_eig_top_r(cases[0][0], 8, ctx=ctx)
    np.testing.assert_array_equal(again.values, results[0].values)
    np.testing.assert_array_equal(again.vectors, results[0].vectors)
