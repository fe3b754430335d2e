"""The register-tile Cholesky + inverse (jacobi.cu chol_inv_tile_kernel,
option chol_reg) against the shared-memory kernel it replaces and LAPACK:
through thin_qr (CholeskyQR3, linalg.hpp:126-149) and the ALS SPD solves
(solvers.hpp:104,109; NotSPD on a non-positive pivot)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture
def cctx():
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    yield ctx
    ctx.set_option("chol_reg", 1)


@pytest.mark.parametrize("m,n", [(50, 1), (300, 3), (1000, 16), (2000, 33), (2048, 80), (3000, 112)])
def test_thin_qr_both_cholesky_kernels(cctx, m, n):
    from paper_2010_10131_b200 import atucker

    rng = np.random.default_rng(m + n)
    a = np.asfortranarray(rng.standard_normal((m, n)) @ np.diag(np.logspace(0, -4, n)))
    q0, r0 = np.linalg.qr(a)
    sg = np.sign(np.diag(r0))
    q0, r0 = q0 * sg, (r0.T * sg).T  # diag(R) >= 0, the reference's normalisation
    out = {}
    for reg in (0, 1):
        cctx.set_option("chol_reg", reg)
        p = atucker.thin_qr(a, ctx=cctx)
        out[reg] = p
        assert np.abs(p.q - q0).max() <= 1e-10
        assert np.abs(p.r - r0).max() <= 1e-12 * np.abs(r0).max()
        assert np.abs(p.q.T @ p.q - np.eye(n)).max() <= 1e-13
    assert np.abs(out[0].q - out[1].q).max() <= 1e-12


def test_als_matches_with_both_cholesky_kernels(cctx):
    from paper_2010_10131_b200 import atucker

    y = np.asfortranarray(np.random.default_rng(4).standard_normal((60, 40, 30)))
    res = {}
    for reg in (0, 1):
        cctx.set_option("chol_reg", reg)
        res[reg] = atucker.als_mode_solver(y, 0, 12, atucker.AlsOptions(num_iters=5, seed=2), ctx=cctx)
    assert np.abs(res[0].factor - res[1].factor).max() <= 1e-11
    assert np.abs(np.asarray(res[0].shrunk) - np.asarray(res[1].shrunk)).max() <= 1e-10 * np.abs(
        np.asarray(res[0].shrunk)).max()


@pytest.mark.parametrize("k", [5, 40, 80, 112])
def test_thin_qr_graded_columns_both_kernels(cctx, k):
    """CholeskyQR3 on columns graded over 1e-7 (the Gram's diagonal spans 1e-14, which the tile
    kernel's unit-diagonal scaling absorbs) and a rank-deficient block (RankDeficient floor,
    linalg.hpp:143-147) with both Cholesky kernels."""
    from paper_2010_10131_b200 import atucker
    from paper_2010_10131_b200.errors import RankDeficient

    rng = np.random.default_rng(k)
    a = np.asfortranarray(rng.standard_normal((3000, k)) * np.logspace(0, -7, k))
    q0, r0 = np.linalg.qr(a)
    sg = np.sign(np.diag(r0))
    q0 = q0 * sg
    for reg in (0, 1):
        cctx.set_option("chol_reg", reg)
        p = atucker.thin_qr(a, ctx=cctx)
        assert np.abs(p.q - q0).max() <= 1e-8
        assert np.abs(p.q.T @ p.q - np.eye(k)).max() <= 1e-13
        if k > 1:
            bad = a.copy()
            bad[:, -1] = bad[:, 0]
            with pytest.raises(RankDeficient):
                atucker.thin_qr(bad, ctx=cctx)
