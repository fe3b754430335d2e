"""The one-pass ALS iteration (csrc/als_tc.cu) against the two-pass schedule
and the CPU oracle.

als_iterate (solvers.hpp:88-118) on mode 0 of an fp32 tensor with R <= 32:
the fused kernel forms rfac = (L^T L)^{-1} L^T Y_(0) tile by tile and feeds it
straight into YR = Y_(0) rfac^T and GR = rfac rfac^T, so Y is read once per
iteration.  Same L0 (mt19937_64 seeding), same update order and NotSPD
checks; results agree with the two-pass path and the oracle to the fp32 bar."""
import numpy as np
import pytest

from conftest import principal_angle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,r", [((256, 64, 128), 16), ((1024, 96, 200), 32), ((128, 4096), 8),
                                    ((384, 50, 33), 20)])
def test_fused_matches_two_pass_and_oracle(dims, r, oracle):
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context(0)
    ctx.set_option("als_gram", 0)  # the passes over Y (the Gram route: test_gram_route_*)
    x = atucker.DeviceTensor.uniform(list(dims), 7, np.float32, ctx=ctx)
    opts = atucker.AlsOptions(seed=3)
    res = {}
    for fused in (1, 0):
        ctx.set_option("als_fused", fused)
        res[fused] = atucker.als_mode_solver(x, 0, r, opts, ctx=ctx)
    f1, f0 = res[1].factor, res[0].factor
    assert np.abs(f1.T @ f1 - np.eye(r)).max() <= 1e-6
    assert principal_angle(f1, f0) <= 2e-3
    g1 = np.linalg.norm(res[1].shrunk.to_numpy().astype(np.float64))
    g0 = np.linalg.norm(res[0].shrunk.to_numpy().astype(np.float64))
    assert abs(g1 - g0) / g0 <= 1e-4
    ref = oracle.als_mode_solver(x.to_numpy().astype(np.float64), 0, r, seed=3)
    gr = np.linalg.norm(ref.shrunk)
    assert abs(g1 - gr) / gr <= 1e-4
    assert principal_angle(f1, ref.factor) <= 2e-3


def test_fused_path_is_taken_and_one_pass():
    """The fused path launches one ALS kernel + one reduction per iteration
    instead of the two-pass TTM / TTM / TTT / Gram chain."""
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context(0)
    ctx.set_option("als_gram", 0)
    x = atucker.DeviceTensor.uniform([512, 64, 64], 9, np.float32, ctx=ctx)
    counts = {}
    for fused in (1, 0):
        ctx.set_option("als_fused", fused)
        l0 = ctx.launch_count
        atucker.als_mode_solver(x, 0, 16, atucker.AlsOptions(seed=1), ctx=ctx)
        counts[fused] = ctx.launch_count - l0
    assert counts[1] < counts[0]


@pytest.mark.parametrize("dims,mode,r", [((1024, 96, 200), 0, 32), ((512, 64, 64), 0, 16), ((40, 600, 300), 1, 24),
                                         ((50, 60, 800), 2, 40)])
def test_gram_route_matches_passes_and_oracle(dims, mode, r, oracle):
    """ALS on the mode's Gram (option als_gram): YR = S M^T and GR = M S M^T are the iterates of
    solvers.hpp:88-118 in exact arithmetic; the factor and the shrunk tensor agree with the
    passes-over-Y schedule and with the fp64 oracle to the fp32 bar, with far fewer launches
    over Y (one Gram, one TTM)."""
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context(0)
    x = atucker.DeviceTensor.uniform(list(dims), 13, np.float32, ctx=ctx)
    opts = atucker.AlsOptions(seed=5)
    res = {}
    try:
        for g in (1, 0):
            ctx.set_option("als_gram", g)
            res[g] = atucker.als_mode_solver(x, mode, r, opts, ctx=ctx)
    finally:
        ctx.set_option("als_gram", 1)
    f1, f0 = res[1].factor, res[0].factor
    assert np.abs(f1.T @ f1 - np.eye(r)).max() <= 1e-6
    assert principal_angle(f1, f0) <= 2e-3
    g1 = np.linalg.norm(res[1].shrunk.to_numpy().astype(np.float64))
    ref = oracle.als_mode_solver(x.to_numpy().astype(np.float64), mode, r, seed=5)
    gr = np.linalg.norm(ref.shrunk)
    assert abs(g1 - gr) / gr <= 1e-4
    assert principal_angle(f1, ref.factor) <= 2e-3
