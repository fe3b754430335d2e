"""Special inputs through st-HOSVD against the oracle (sthosvd.hpp:126-194), every solver per mode:
an all-zero tensor, a constant tensor (every unfolding has rank 1 and its rows are exact multiples
of one vector: the one-sided Jacobi SVD must stop rotating them), a single element, a rank-1
tensor, and fp64 data scaled by 1e+-140 (the Gram's entries are then ~1e+-280: the eigensolvers
scale by a power of two first, as Eigen's SelfAdjointEigenSolver does, linalg.hpp:113-126).

Where the oracle itself stops (a Cholesky breakdown in ALS on rank-deficient data,
linalg.hpp:169-177), the engine must stop too; otherwise the core norm agrees to 1e-10 (fp64) /
1e-4 (fp32) and every factor is orthonormal.
"""
import numpy as np
import pytest

from conftest import orthonormality_defect
from test_gpu_sweep import _PerMode

pytestmark = pytest.mark.gpu


def _inputs():
    return {
        "zeros": np.zeros((20, 30, 40)),
        "const": np.full((20, 30, 40), 3.0),
        "one": np.full((1, 1, 1), 2.0),
        "rank1": np.einsum("i,j,k->ijk", np.arange(1, 21.0), np.ones(30), np.linspace(1, 2, 40)),
        "huge": np.random.default_rng(0).standard_normal((20, 30, 40)) * 1e140,
        "tiny": np.random.default_rng(1).standard_normal((20, 30, 40)) * 1e-140,
    }


_CASES = [(name, kinds, dt) for name in ("zeros", "const", "one", "rank1", "huge", "tiny")
          for kinds in ((0, 0, 0), (1, 1, 1), (2, 2, 2), (0, 1, 2))
          for dt in ("f64", "f32") if not (dt == "f32" and name in ("huge", "tiny"))]


@pytest.mark.parametrize("name,kinds,dt", _CASES)
def test_special_input(name, kinds, dt, oracle):
    from paper_2010_10131_b200 import atucker

    x = _inputs()[name]
    dtype = np.float64 if dt == "f64" else np.float32
    xx = np.asfortranarray(x.astype(dtype))
    ranks = [min(3, d) for d in x.shape]
    try:
        ref = oracle.sthosvd(xx.astype(np.float64), ranks, lambda m, i, r, j: kinds[m], seed=1)
    except Exception:  # noqa: BLE001 - the oracle's own stop (Cholesky breakdown)
        with pytest.raises(Exception):
            atucker.sthosvd(xx, ranks, _PerMode(list(kinds)), atucker.AlsOptions(seed=1))
        return
    res = atucker.sthosvd(xx, ranks, _PerMode(list(kinds)), atucker.AlsOptions(seed=1))
    core = np.asarray(res.decomposition.core, dtype=np.float64)
    assert np.all(np.isfinite(core))
    g, gr = np.linalg.norm(core), np.linalg.norm(ref.core)
    tol = 1e-10 if dtype == np.float64 else 1e-4
    assert abs(g - gr) <= tol * gr or g == gr, (g, gr)
    for f in res.decomposition.factors:
        assert orthonormality_defect(f) <= (1e-10 if dtype == np.float64 else 1e-5)


@pytest.mark.parametrize("scale", [1e150, 1e-150])
@pytest.mark.parametrize("n,method", [(60, -1), (400, 1), (300, 3)])
def test_sym_eig_scaled(scale, n, method, oracle):
    """The eigensolver alone on a Gram scaled far outside fp64's comfortable range: values scale
    exactly (a power of two round trip), vectors unchanged."""
    from paper_2010_10131_b200 import atucker

    rng = np.random.default_rng(n)
    q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    lam = np.linspace(n, 1, n)
    s = (q * lam) @ q.T
    ctx = atucker.Context.default(0)
    ctx.set_option("eig_method", method)
    try:
        p0 = atucker.sym_eig_top_r(s, 8, ctx=ctx)
        p1 = atucker.sym_eig_top_r(s * scale, 8, ctx=ctx)
    finally:
        ctx.set_option("eig_method", -1)
    v0, v1 = p0.values, p1.values
    assert np.all(np.isfinite(v1))
    np.testing.assert_allclose(v1 / scale, v0, rtol=1e-12)
    np.testing.assert_allclose(np.abs(p1.vectors), np.abs(p0.vectors), atol=1e-10)
