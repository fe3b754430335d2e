"""Parity at the full BASELINE sizes (C2 1024^3, C5 2048^3, fp32).

The oracle runs on the GPU box's host cores on the very bytes the engine
consumed (device-generated input copied back).  C5 uses the oracle's
memory-lean fp32 entry (mode-0 Gram/TTM streamed in fp64 chunks) because
the fp64 copy of 2048^3 alone is 69 GB.  Criteria:
core-norm relative difference <= 1e-4, |relative-error difference| <= 1e-4,
principal angles <= 1e-3 on the gapped C5 input, orthonormal factors.
The relative error of the EIG strategy is checked through the projection
identity ||X - Xhat||^2 = ||X||^2 - ||G||^2 (exact for orthonormal factors
when every mode is an EIG/SVD projection).
"""
import os

import numpy as np
import pytest

from conftest import orthonormality_defect, principal_angle
from paper_2010_10131_b200.selector import SolverKind, Strategy

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def test_c5_full_2048_cubed(oracle, capsys):
    import bench
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    cfg = bench.CONFIGS["c5"]
    x = bench.make_input(atucker, cfg, bench.SEEDS["c5"], ctx)
    res = atucker.sthosvd(x, cfg["ranks"], Strategy.fixed_eig(), ctx=ctx)
    core = res.decomposition.core.to_numpy().astype(np.float64)
    # engine side: the true ||X - Xhat|| / ||X|| by reconstruction on the device
    # (the projection identity only holds for an exact fp64 projection: with the
    # low 1e-2 noise, eps^2 ~ 1e-4 would amplify the tf32 core error 1e4-fold)
    e_gpu = atucker.relative_error(x, res.decomposition, ctx=ctx)
    xh = x.to_numpy()
    x.free()
    ref = oracle.sthosvd_f32_eig0(xh, cfg["ranks"], threads=os.cpu_count() or 8)
    nx2 = oracle.norm2_f32(xh)
    del xh
    g, gr = np.linalg.norm(core), np.linalg.norm(ref.core)
    e_cpu = np.sqrt(max(0.0, 1.0 - gr * gr / nx2))  # exact for the oracle's fp64 projections
    angles = [principal_angle(a, b) for a, b in zip(res.decomposition.factors, ref.factors)]
    with capsys.disabled():
        print(f"\nC5 full: |G| gpu {g:.9e} cpu {gr:.9e} rel {abs(g - gr) / gr:.2e}; "
              f"err gpu {e_gpu:.6e} cpu {e_cpu:.6e}; max angle {max(angles):.2e}")
    assert abs(g - gr) / gr <= 1e-4
    assert abs(e_gpu - e_cpu) <= 1e-4
    assert max(angles) <= 1e-3
    for f in res.decomposition.factors:
        assert orthonormality_defect(f) <= 1e-10


def test_c2_full_1024_cubed_mixed(oracle, capsys):
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    xd = atucker.DeviceTensor.uniform([1024, 1024, 1024], 2, np.float32, ctx=ctx)
    s = Strategy.manual([SolverKind.Als, SolverKind.Eig, SolverKind.Eig])
    res = atucker.sthosvd(xd, [32, 32, 32], s, ctx=ctx)
    core = res.decomposition.core.to_numpy().astype(np.float64)
    xh = xd.to_numpy()
    xd.free()
    oracle.set_threads(os.cpu_count() or 8)
    x64 = xh.astype(np.float64)
    del xh
    ref = oracle.sthosvd(x64, [32, 32, 32], lambda m, i, r, j: int(s.decide(m, i, r, j)))
    g, gr = np.linalg.norm(core), np.linalg.norm(ref.core)
    e_gpu = atucker.relative_error(x64, res.decomposition, ctx=ctx)
    e_cpu = oracle.relative_error(x64, ref.core, ref.factors)
    with capsys.disabled():
        print(f"\nC2 full: |G| gpu {g:.9e} cpu {gr:.9e} rel {abs(g - gr) / gr:.2e}; "
              f"err gpu {e_gpu:.6e} cpu {e_cpu:.6e}")
    assert abs(g - gr) / gr <= 1e-4
    assert abs(e_gpu - e_cpu) <= 1e-4
    for f in res.decomposition.factors:
        assert orthonormality_defect(f) <= 1e-10


def test_c5u_full_2048_cubed(oracle, capsys):
    """SURVEY §8(d) C5 stress row: uniform 2048^3 (flat Marchenko-Pastur Gram
    spectra, the 64 wanted eigenvalues within 0.6% of each other) through the
    default dispatch (ChFSI handing over to the exact dense solver).  Core norm
    and relative error within 1e-4 of the oracle; the factors' subspaces are
    ill-determined at tf32 Gram accuracy on a flat spectrum, so they are
    checked for orthonormality only."""
    import bench
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    cfg = bench.CONFIGS["c5u"]
    x = bench.make_input(atucker, cfg, bench.SEEDS["c5u"], ctx)
    res = atucker.sthosvd(x, cfg["ranks"], Strategy.fixed_eig(), ctx=ctx)
    core = res.decomposition.core.to_numpy().astype(np.float64)
    e_gpu = atucker.relative_error(x, res.decomposition, ctx=ctx)
    xh = x.to_numpy()
    x.free()
    ref = oracle.sthosvd_f32_eig0(xh, cfg["ranks"], threads=os.cpu_count() or 8)
    nx2 = oracle.norm2_f32(xh)
    del xh
    g, gr = np.linalg.norm(core), np.linalg.norm(ref.core)
    e_cpu = np.sqrt(max(0.0, 1.0 - gr * gr / nx2))
    with capsys.disabled():
        print(f"\nC5u full: |G| gpu {g:.9e} cpu {gr:.9e} rel {abs(g - gr) / gr:.2e}; "
              f"err gpu {e_gpu:.9e} cpu {e_cpu:.9e}; eig methods {[r.eig_method for r in res.reports]}")
    assert abs(g - gr) / gr <= 1e-4
    assert abs(e_gpu - e_cpu) <= 1e-4
    for f in res.decomposition.factors:
        assert orthonormality_defect(f) <= 1e-10
