"""The tridiagonal dense eigensolver (csrc/tridiag.cu) against LAPACK.

linalg::sym_eig_top_r (linalg.hpp:101-123) keeps the top r eigenpairs,
descending, sign-fixed.  The engine's default for n <= 200 reduces to
tridiagonal form (Householder), finds the wanted eigenvalues by Sturm
bisection and their vectors by inverse iteration with in-cluster
Gram-Schmidt (the dsytrd/dstebz/dstein structure).  Checked here on spectra
that stress each stage: flat (everything clustered), exactly degenerate,
rank-deficient (zero cluster), indefinite, graded over 12 decades, tiny n.

Bars: eigenvalues 1e-12 relative to ||A||; residual ||A V - V diag(w)|| and
orthonormality 1e-11 (both hold for every returned vector, clustered or not);
vectors of well-separated eigenvalues within 1e-9 (principal angle) of LAPACK.
"""
import numpy as np
import pytest

from conftest import orthonormality_defect, principal_angle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tctx():
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context(0)
    ctx.set_option("eig_method", 2)
    return ctx


def _spectrum_matrix(n, lam, seed):
    rng = np.random.default_rng(seed)
    q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    s = (q * lam) @ q.T
    return (s + s.T) / 2


def _check(s, r, res):
    w_all, q_all = np.linalg.eigh(s)
    w, q = w_all[::-1][:r], q_all[:, ::-1][:, :r]
    scale = max(np.abs(w_all).max(), 1e-300)
    assert np.abs(res.values - w).max() <= 1e-12 * scale
    v = res.vectors
    assert orthonormality_defect(v) <= 1e-11
    assert np.abs(s @ v - v * res.values).max() <= 1e-11 * scale
    for j in range(r):
        c = v[:, j]
        assert c[np.argmax(np.abs(c))] > 0
    full = w_all[::-1]
    for j in range(r):
        gap = min(abs(full[j] - full[j - 1]) if j > 0 else np.inf,
                  abs(full[j] - full[j + 1]) if j + 1 < len(full) else np.inf)
        if gap > 1e-6 * scale:
            assert principal_angle(v[:, j:j + 1], q[:, j:j + 1]) <= 1e-9


@pytest.mark.parametrize("n", [1, 2, 3, 7, 31, 32, 33, 64, 96, 127, 160, 192, 193, 197, 200])
def test_random_symmetric(tctx, n):
    from paper_2010_10131_b200 import atucker

    rng = np.random.default_rng(100 + n)
    b = rng.standard_normal((n, n))
    s = (b + b.T) / 2
    r = max(1, (2 * n) // 3)
    _check(s, r, atucker.sym_eig_top_r(s, r, ctx=tctx))


@pytest.mark.parametrize("n", [48, 128, 200])
def test_flat_gram(tctx, n):
    """Marchenko-Pastur Gram (the C1 shape): every wanted value is in a cluster."""
    from paper_2010_10131_b200 import atucker

    rng = np.random.default_rng(n)
    a = rng.standard_normal((n, 40 * n))
    s = a @ a.T
    _check(s, n // 2, atucker.sym_eig_top_r(s, n // 2, ctx=tctx))


@pytest.mark.parametrize("n", [193, 200])
def test_short_tile_row_matches_column_kernel(tctx, n):
    """192 < n <= 200 runs the tile reduction with a short 7th tile row (trd_tile_kernel<7>); the
    column-slot kernel (option trd_tiles 0) is an independent implementation of the same dsytd2
    reduction: same eigenvalues, same subspaces, on a graded spectrum."""
    from paper_2010_10131_b200 import atucker

    s = _spectrum_matrix(n, np.logspace(4, -4, n), 7)
    r = n // 3
    tiles = atucker.sym_eig_top_r(s, r, ctx=tctx)
    ctx2 = atucker.Context(0)
    ctx2.set_option("trd_tiles", 0)
    cols = atucker.sym_eig_top_r(s, r, ctx=ctx2)
    np.testing.assert_allclose(tiles.values, cols.values, rtol=1e-12, atol=1e-12 * abs(cols.values[0]))
    _check(s, r, tiles)
    for j in range(r):
        assert principal_angle(tiles.vectors[:, j:j + 1], cols.vectors[:, j:j + 1]) <= 1e-9


def test_all_wanted_flat_spectrum(tctx):
    """nwant = n on a flat spectrum: one cluster of n members."""
    from paper_2010_10131_b200 import atucker

    n = 96
    s = _spectrum_matrix(n, 1.0 + 1e-4 * np.random.default_rng(1).random(n), 2)
    _check(s, n, atucker.sym_eig_top_r(s, n, ctx=tctx))


@pytest.mark.parametrize("mult", [2, 5, 40])
def test_degenerate(tctx, mult):
    from paper_2010_10131_b200 import atucker

    n = 80
    lam = np.concatenate([np.full(mult, 3.0), np.linspace(2.0, 0.5, n - mult)])
    s = _spectrum_matrix(n, lam, mult)
    res = atucker.sym_eig_top_r(s, mult + 4, ctx=tctx)
    _check(s, mult + 4, res)
    # the degenerate block: any orthonormal basis of the eigenspace
    q = np.linalg.eigh(s)[1][:, ::-1][:, :mult]
    assert principal_angle(res.vectors[:, :mult], q) <= 1e-9


def test_identity_and_zero(tctx):
    from paper_2010_10131_b200 import atucker

    for s in (np.eye(20), np.zeros((20, 20))):
        _check(s, 7, atucker.sym_eig_top_r(s, 7, ctx=tctx))


def test_rank_deficient(tctx):
    from paper_2010_10131_b200 import atucker

    a = np.random.default_rng(3).standard_normal((150, 12))
    s = a @ a.T
    _check(s, 20, atucker.sym_eig_top_r(s, 20, ctx=tctx))  # 8 of 20 in the zero cluster


def test_graded(tctx):
    from paper_2010_10131_b200 import atucker

    n = 120
    s = _spectrum_matrix(n, np.logspace(6, -6, n), 9)
    _check(s, 40, atucker.sym_eig_top_r(s, 40, ctx=tctx))


def test_already_tridiagonal_and_diagonal(tctx):
    from paper_2010_10131_b200 import atucker

    n = 64
    d = np.linspace(1, 2, n)
    t = np.diag(d) + np.diag(np.full(n - 1, 0.3), 1) + np.diag(np.full(n - 1, 0.3), -1)
    _check(t, 10, atucker.sym_eig_top_r(t, 10, ctx=tctx))
    _check(np.diag(d[::-1].copy()), 10, atucker.sym_eig_top_r(np.diag(d[::-1].copy()), 10, ctx=tctx))


def test_bit_reproducible(tctx):
    """No atomics anywhere: sharded ranks rely on bit-identical factors."""
    from paper_2010_10131_b200 import atucker

    a = np.random.default_rng(4).standard_normal((200, 900))
    s = a @ a.T
    r1 = atucker.sym_eig_top_r(s, 20, ctx=tctx)
    r2 = atucker.sym_eig_top_r(s, 20, ctx=tctx)
    np.testing.assert_array_equal(r1.values, r2.values)
    np.testing.assert_array_equal(r1.vectors, r2.vectors)


@pytest.mark.parametrize("variant", [1, 2, 0], ids=["warps", "tiles", "slots"])
@pytest.mark.parametrize("n", [5, 32, 33, 48, 64, 80, 97, 128])
def test_reduction_kernels(variant, n):
    """The three Householder reductions (option trd_tiles): 1 = one to four
    warps for n <= 128 (the default), 2 = the 32 x 32 tile kernel, 0 = the
    column-slot kernel.  Same outputs, same bars."""
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context(0)
    ctx.set_option("eig_method", 2)
    ctx.set_option("trd_tiles", variant)
    try:
        rng = np.random.default_rng(7 * n + variant)
        a = rng.standard_normal((n, 3 * n))
        s = a @ a.T
        _check(s, max(1, n // 2), atucker.sym_eig_top_r(s, max(1, n // 2), ctx=ctx))
        b = rng.standard_normal((n, n))
        _check((b + b.T) / 2, n, atucker.sym_eig_top_r((b + b.T) / 2, n, ctx=ctx))
    finally:
        ctx.set_option("trd_tiles", 1)
        ctx.set_option("eig_method", -1)


@pytest.mark.parametrize("n,kind", [(80, "gram"), (80, "flat"), (128, "flat"), (48, "degenerate")])
def test_invit_shared_memory_variant_bit_identical(n, kind):
    """Inverse iteration with its working set in shared memory (option invit_smem, the default for
    n <= 128) does the same arithmetic in the same order as the global-memory kernel: the vectors are
    bit-identical, including clusters of more than 32 members (the flat spectra: one chunk of 32
    in shared memory, earlier chunks read back from the output)."""
    from paper_2010_10131_b200 import atucker

    rng = np.random.default_rng(n)
    if kind == "gram":
        a = rng.standard_normal((n, 3 * n))
        s = a @ a.T
    elif kind == "flat":
        s = _spectrum_matrix(n, 1.0 + 1e-9 * rng.standard_normal(n), n)
    else:
        s = _spectrum_matrix(n, np.repeat([3.0, 2.0, 1.0], [20, 20, n - 40]), n)
    ctx = atucker.Context(0)
    ctx.set_option("eig_method", 2)
    out = {}
    try:
        for v in (1, 0):
            ctx.set_option("invit_smem", v)
            out[v] = atucker.sym_eig_top_r(s, n - 4, ctx=ctx)
    finally:
        ctx.set_option("invit_smem", 1)
    np.testing.assert_array_equal(out[0].values, out[1].values)
    np.testing.assert_array_equal(out[0].vectors, out[1].vectors)
    _check(s, n - 4, out[1])
