"""Parity of the CUDA engine with the CPU oracle on the BASELINE configs.

Same input bytes on both sides (device-generated fp32 inputs are copied back
for the oracle).  Criteria:
  core-norm relative difference   <= 1e-10 (fp64) / 1e-4 (fp32)
  |relative error difference|     <= 1e-10 (fp64) / 1e-4 (fp32)
  principal angles per factor     <= 1e-8 (fp64) / 1e-3 (fp32), gapped inputs only
  factor orthonormality           <= 1e-10
Full-size C2/C5 are checked through size-independent properties (the
orthogonal-projection identity ||X - Xhat||^2 = ||X||^2 - ||G||^2 for EIG
strategies) in test_gpu_fullsize.py and bench.py.
"""
import os

import numpy as np
import pytest

from conftest import orthonormality_defect, principal_angle
from paper_2010_10131_b200.selector import SolverKind, Strategy

pytestmark = pytest.mark.gpu


def _threads():
    import oracle as o

    o.set_threads(os.cpu_count() or 8)


def _compare(x_host, res, ref, tol_norm, tol_err, tol_angle=None):
    import oracle as o
    from paper_2010_10131_b200 import atucker

    core = res.decomposition.core
    core = core.to_numpy() if isinstance(core, atucker.DeviceTensor) else core
    g_gpu = np.linalg.norm(core.astype(np.float64))
    g_cpu = np.linalg.norm(ref.core)
    assert abs(g_gpu - g_cpu) / g_cpu <= tol_norm, (g_gpu, g_cpu)
    for f in res.decomposition.factors:
        assert orthonormality_defect(f) <= 1e-10
    e_cpu = o.relative_error(x_host, ref.core, ref.factors)
    e_gpu = atucker.relative_error(x_host, res.decomposition)
    assert abs(e_gpu - e_cpu) <= tol_err, (e_gpu, e_cpu)
    if tol_angle is not None:
        for fg, fc in zip(res.decomposition.factors, ref.factors):
            assert principal_angle(fg, fc) <= tol_angle
    return e_gpu, e_cpu


def test_c1_reference_input_fixed_eig(oracle):
    """C1: 200^3 fp64, ranks 20^3, EIG every mode, the reference's own input
    random_tensor({200,200,200}, 1, StandardNormal) (golden-pinned)."""
    from paper_2010_10131_b200 import atucker

    _threads()
    x = oracle.random_tensor([200, 200, 200], 1, "normal")
    ref = oracle.sthosvd(x, [20, 20, 20])
    res = atucker.sthosvd(x, [20, 20, 20], Strategy.fixed_eig())
    _compare(x, res, ref, 1e-10, 1e-10)


def test_c1_lowrank_angles(oracle):
    """C1 gapped variant: synth_lowrank(200^3, 20^3) + 1e-2 noise -> factor-level parity."""
    from paper_2010_10131_b200 import atucker

    _threads()
    x = oracle.synth_lowrank([200, 200, 200], [20, 20, 20], 2024)
    x = x + 1e-2 * oracle.random_tensor([200, 200, 200], 7, "normal")
    ref = oracle.sthosvd(x, [20, 20, 20])
    res = atucker.sthosvd(x, [20, 20, 20], Strategy.fixed_eig())
    _compare(x, res, ref, 1e-10, 1e-10, tol_angle=1e-8)
    for fg, fc in zip(res.decomposition.factors, ref.factors):
        assert np.abs(fg - fc).max() <= 1e-8  # sign rule makes factors entry-wise comparable


def test_c1_costmodel_strategy(oracle):
    """C1 under the reference cost model (picks e,e,a): same decisions, same ALS start."""
    from paper_2010_10131_b200 import atucker
    from paper_2010_10131_b200.selector import CostModelParams

    _threads()
    x = oracle.random_tensor([200, 200, 200], 1, "normal")
    s = Strategy.cost_model()
    p = CostModelParams()
    ref = oracle.sthosvd(x, [20, 20, 20], lambda m, i, r, j: int(s.decide(m, i, r, j, p)))
    res = atucker.sthosvd(x, [20, 20, 20], s)
    assert [int(r.solver_used) for r in res.reports] == [int(v) for v in ref.reports[:, 0]]
    assert [int(r.solver_used) for r in res.reports] == [0, 0, 1]
    _compare(x, res, ref, 1e-10, 1e-10)


def test_c3_four_way_fp64(oracle):
    """C3: 128^4 fp64, ranks 16^4, EIG every mode (non-contiguous middle modes)."""
    from paper_2010_10131_b200 import atucker

    _threads()
    x = oracle.random_tensor([128, 128, 128, 128], 3, "normal")
    ref = oracle.sthosvd(x, [16, 16, 16, 16])
    res = atucker.sthosvd(x, [16, 16, 16, 16], Strategy.fixed_eig())
    _compare(x, res, ref, 1e-10, 1e-10)


def test_c4_five_way_fp32(oracle):
    """C4: 48^5 fp32 counter-hash uniform (seed 4), ranks 8^5, EIG every mode."""
    from paper_2010_10131_b200 import atucker

    _threads()
    xd = atucker.DeviceTensor.uniform([48] * 5, 4, np.float32)
    xh = xd.to_numpy()
    np.testing.assert_array_equal(xh.ravel(order="F")[:4096], oracle.hash_uniform(4, 4096))
    ref = oracle.sthosvd(xh.astype(np.float64), [8] * 5)
    res = atucker.sthosvd(xd, [8] * 5, Strategy.fixed_eig())
    _compare(xh.astype(np.float64), res, ref, 1e-4, 1e-4)


def test_c2_mixed_reduced(oracle):
    """C2 shape family at 256^3 (full 1024^3 in test_gpu_fullsize): fp32 uniform,
    ranks 32^3, canonical manual:a,e,e (ALS on mode 1 with the reference L0)."""
    from paper_2010_10131_b200 import atucker

    _threads()
    xd = atucker.DeviceTensor.uniform([256, 256, 256], 2, np.float32)
    xh = xd.to_numpy().astype(np.float64)
    s = Strategy.manual([SolverKind.Als, SolverKind.Eig, SolverKind.Eig])
    ref = oracle.sthosvd(xh, [32, 32, 32], lambda m, i, r, j: int(s.decide(m, i, r, j)))
    res = atucker.sthosvd(xd, [32, 32, 32], s)
    _compare(xh, res, ref, 1e-4, 1e-4)


def test_c5_lowrank_reduced(oracle):
    """C5 shape family at 512^3 (full 2048^3 in test_gpu_fullsize / bench):
    low-rank 64^3 core + 1e-2 noise, ranks 64^3, EIG (ChFSI eig at n = 512)."""
    from paper_2010_10131_b200 import atucker

    _threads()
    xd = lowrank_plus_noise([512, 512, 512], [64, 64, 64], 5)
    xh = xd.to_numpy().astype(np.float64)
    ref = oracle.sthosvd(xh, [64, 64, 64])
    res = atucker.sthosvd(xd, [64, 64, 64], Strategy.fixed_eig())
    _compare(xh, res, ref, 1e-4, 1e-4, tol_angle=1e-3)


def lowrank_plus_noise(dims, ranks, seed, noise=1e-2, dtype=np.float32):
    """Device generator of the canonical C5 input: a uniform core expanded by
    orthonormal factors (reconstruct on the device) + noise * uniform."""
    from paper_2010_10131_b200 import atucker
    import oracle as o

    rng = np.random.default_rng(seed)
    core = atucker.DeviceTensor.uniform(ranks, seed, dtype)
    factors = [np.linalg.qr(rng.standard_normal((d, r)))[0] for d, r in zip(dims, ranks)]
    t = atucker.TuckerDecomposition(core, factors, tuple(dims))
    x = atucker.reconstruct(t)
    scale = np.sqrt(np.prod(dims) / np.prod(ranks))  # signal entries ~ O(1)
    nz = atucker.DeviceTensor.uniform(dims, seed + 1000, dtype)
    x.axpy(scale - 1.0, x)  # x <- scale * x
    x.axpy(noise, nz)       # x <- x + noise * uniform
    nz.free()
    return x


def test_frobenius_norm_device_fp32_large():
    """atk_frobenius_norm (tensor.hpp:158-168) on a 64M-element fp32 device tensor
    (the counter-hash stream, bit-identical to the oracle's), accumulated in fp64."""
    import sys
    from pathlib import Path

    from paper_2010_10131_b200 import atucker

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "oracle"))
    import oracle as o

    ctx = atucker.Context.default(0)
    dims = [512, 512, 256]
    x = atucker.DeviceTensor.uniform(dims, 21, np.float32, ctx=ctx)
    ref = np.sqrt(o.norm2_f32(o.hash_uniform(21, int(np.prod(dims)))))
    got = atucker.frobenius_norm(x, ctx=ctx)
    # the oracle sums 64M squares serially in fp64 (its own error ~sqrt(n) eps ~ 1e-12);
    # an fp32 accumulation would be off by ~1e-4
    assert abs(got - ref) <= 1e-10 * ref, (got, ref)


@pytest.mark.parametrize("dims,mode", [([128, 40, 30], 0), ([31, 7, 9], 0), ([20, 30, 192], 2), ([6, 5, 97], 2),
                                       ([64, 3000], 0), ([160, 50, 4], 0), ([200, 50, 4], 0)])
def test_fp64_first_last_mode_gram_syrk(dims, mode):
    """The fp64 first / last-mode Gram (kernels.hpp:127-138) runs as a SYRK on DMMA (dgemm.cu
    syrk_panel_kernel, n <= 160; n = 200 keeps the GEMM): exactly symmetric, and equal to the
    fp64 product to rounding."""
    from paper_2010_10131_b200 import atucker

    x = np.asfortranarray(np.random.default_rng(sum(dims)).standard_normal(dims))
    g = atucker.gram(x, mode)
    m = np.moveaxis(x, mode, 0).reshape(dims[mode], -1, order="F")
    want = m @ m.T
    np.testing.assert_array_equal(g, g.T)
    assert np.abs(g - want).max() <= 1e-12 * np.abs(want).max()


@pytest.mark.parametrize("dims,mode,r", [([128, 40, 30], 0, 16), ([31, 7, 9], 0, 5), ([20, 30, 40], 2, 33),
                                         ([6, 5, 97], 2, 64), ([200, 500], 0, 20), ([64, 3000], 1, 1)])
def test_fp64_first_last_mode_ttm_gemm(dims, mode, r):
    """The fp64 first / last-mode TTM (kernels.hpp:88-118) on the pipelined DMMA GEMM (dgemm.cu
    dgemm_ttm; mode 0 stores the transposed product): equal to the fp64 product to rounding."""
    from paper_2010_10131_b200 import atucker

    rng = np.random.default_rng(sum(dims) + r)
    x = np.asfortranarray(rng.standard_normal(dims))
    u = rng.standard_normal((r, dims[mode]))
    y = atucker.ttm(x, u, mode)
    y = y.to_numpy() if hasattr(y, "to_numpy") else np.asarray(y)
    want = np.moveaxis(np.tensordot(u, x, axes=([1], [mode])), 0, mode)
    assert y.shape == want.shape
    assert np.abs(y - want).max() <= 1e-12 * np.abs(want).max()


def test_large_rank_als_and_thin_qr(oracle):
    """Ranks beyond the one-CTA Cholesky (k <= 112): thin_qr of 200 columns through the Householder
    kernel (linalg.hpp:126-149), and an ALS mode with R = 150 (solvers.hpp:88-138), against the
    oracle / LAPACK."""
    from paper_2010_10131_b200 import atucker

    rng = np.random.default_rng(21)
    a = np.asfortranarray(rng.standard_normal((600, 200)))
    p = atucker.thin_qr(a)
    q0, r0 = np.linalg.qr(a)
    sg = np.sign(np.diag(r0))
    assert np.abs(p.q - q0 * sg).max() <= 1e-10
    assert np.abs(p.q.T @ p.q - np.eye(200)).max() <= 1e-12
    y = np.asfortranarray(rng.standard_normal((300, 40, 40)))
    res = atucker.als_mode_solver(y, 0, 150, atucker.AlsOptions(num_iters=3, seed=4))
    ref = oracle.als_mode_solver(y, 0, 150, num_iters=3, seed=4)
    assert principal_angle(res.factor, ref.factor) <= 1e-8
    assert abs(np.linalg.norm(np.asarray(res.shrunk)) - np.linalg.norm(ref.shrunk)) <= 1e-10 * np.linalg.norm(ref.shrunk)
