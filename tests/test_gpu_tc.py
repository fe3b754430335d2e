"""tcgen05 (kind::tf32) Gram kernel vs the fp64 oracle, all operand layouts.

tf32 keeps 10 mantissa bits, so the Gram is compared with a relative bound
of 4e-3 on max|dS| / max|S| (exactly symmetric output is still required).  The
test also records which tf32 conversion the hardware applies (truncation vs
round-to-nearest) by comparing against both emulations in fp64.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def tf32_trunc(x):
    b = np.asarray(x, dtype=np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return b.view(np.float32).astype(np.float64)


def tf32_rn(x):
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return u.view(np.float32).astype(np.float64)


def gram_np(x, n):
    m = np.moveaxis(x, n, 0).reshape(x.shape[n], -1, order="F")
    return m @ m.T


@pytest.mark.parametrize("dims,mode", [
    ((256, 1000), 0), ((300, 64, 7), 0), ((1024, 2048), 0), ((128, 4096), 0),   # MN-major (mode 0)
    ((32, 256, 40), 1), ((64, 512, 9), 1), ((4096, 300), 1), ((96, 200, 5), 1),  # K-major (P >= 32)
    ((48, 9000), 0), ((32, 20000), 0), ((8, 4000), 0), ((48, 48, 300), 1),       # small I: half-width tile
    ((8, 48, 301), 1), ((16, 40, 77), 1), ((4, 64, 50, 3), 1), ((8, 300, 61), 1),  # P in {4, 8, 16}: 16-B panels
])
@pytest.mark.parametrize("tma_tf32", [0, 1])
def test_tc_gram_vs_oracle(dims, mode, tma_tf32, capsys):
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    ctx.set_option("tma_tf32", tma_tf32)
    xd = atucker.DeviceTensor.uniform(list(dims), 11, np.float32)
    x = xd.to_numpy()
    launches = ctx.launch_count
    s = atucker.gram(xd, mode)
    assert ctx.launch_count - launches == 2  # gram_tf32_kernel + gram_reduce
    ref = gram_np(x.astype(np.float64), mode)
    scale = np.abs(ref).max()
    err = np.abs(s - ref).max() / scale
    assert np.array_equal(s, s.T)
    assert err <= 4e-3, err
    et = np.abs(s - gram_np(tf32_trunc(x), mode)).max() / scale
    er = np.abs(s - gram_np(tf32_rn(x), mode)).max() / scale
    d = np.diag(s) / np.diag(ref) - 1.0
    with capsys.disabled():
        print(f"\nTF32MODE dims={dims} mode={mode} tma_tf32={tma_tf32} err={err:.2e} "
              f"vs_trunc={et:.2e} vs_rn={er:.2e} diag_bias={d.mean():+.2e}")
    ctx.set_option("tma_tf32", 1)  # restore the engine default (RN tf32 via TMA)


def test_tc_gram_long_k_chunked():
    """Long K (fp32 chains bounded by the fp64 drains): diagonal bias stays small."""
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    xd = atucker.DeviceTensor.uniform([128, 1 << 20], 3, np.float32)
    x = xd.to_numpy().astype(np.float64)
    s = atucker.gram(xd, 0)
    ref = x @ x.T
    err = np.abs(s - ref).max() / np.abs(ref).max()
    assert err <= 4e-3


@pytest.mark.parametrize("dims,mode,r", [
    ((256, 1000), 0, 64), ((300, 64, 7), 0, 20), ((2048, 777), 0, 128), ((96, 40, 3), 0, 33),  # K-major A
    ((64, 256, 9), 1, 64), ((32, 128, 5), 1, 32), ((4096, 96), 1, 16), ((64, 64, 64), 2, 64),  # MN-major A
    ((64, 64, 2048), 2, 64), ((64, 2048, 100), 1, 64), ((96, 128, 40), 1, 24),  # 4-D / 3-D boxes, split-K
    ((128, 512, 2), 1, 32),
])
def test_tc_ttm_vs_oracle(dims, mode, r, capsys):
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    xd = atucker.DeviceTensor.uniform(list(dims), 13, np.float32)
    x = xd.to_numpy().astype(np.float64)
    rng = np.random.default_rng(5)
    u = np.linalg.qr(rng.standard_normal((dims[mode], r)))[0].T.copy(order="F")  # R x I, orthonormal rows
    launches = ctx.launch_count
    y = atucker.ttm(xd, u, mode).to_numpy().astype(np.float64)
    n_launch = ctx.launch_count - launches
    ref = np.moveaxis(np.tensordot(u, x, axes=([1], [mode])), 0, mode)
    err = np.abs(y - ref).max() / np.abs(ref).max()
    nrm = abs(np.linalg.norm(y) - np.linalg.norm(ref)) / np.linalg.norm(ref)
    with capsys.disabled():
        print(f"\nTTM dims={dims} mode={mode} r={r} launches={n_launch} maxrel={err:.2e} normrel={nrm:.2e}")
    assert err <= 4e-3 and nrm <= 1e-4
    assert n_launch in (2, 3)  # factor cast + ttm_tf32_kernel (+ the split-K reduction)


@pytest.mark.parametrize("dims,mode", [
    ((512, 5000), 0), ((2048, 1000), 0), ((768, 33, 20), 0),   # MN-major, CTA pairs
    ((64, 1024, 5), 1), ((32, 768, 40), 1), ((256, 2048), 1),  # K-major, CTA pairs
])
def test_tc_gram_2cta_matches_1cta_and_oracle(dims, mode, capsys):
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    xd = atucker.DeviceTensor.uniform(list(dims), 17, np.float32)
    x = xd.to_numpy().astype(np.float64)
    ctx.set_option("gram_2cta", 1)
    s2 = atucker.gram(xd, mode)
    ctx.set_option("gram_2cta", 0)
    s1 = atucker.gram(xd, mode)
    ctx.set_option("gram_2cta", 1)
    ref = gram_np(x, mode)
    scale = np.abs(ref).max()
    e2 = np.abs(s2 - ref).max() / scale
    e1 = np.abs(s1 - ref).max() / scale
    with capsys.disabled():
        print(f"\nGRAM2 dims={dims} mode={mode} err2={e2:.2e} err1={e1:.2e} diff={np.abs(s2 - s1).max() / scale:.2e}")
    assert np.array_equal(s2, s2.T)
    assert e2 <= 1e-4 and e1 <= 1e-4  # RN tf32 (TMA TFLOAT32)


@pytest.mark.parametrize("dims,mode", [((2048, 20000), 0), ((64, 2048, 300), 1)])
def test_tc_gram_2cta_k_launches(dims, mode):
    """The 2-CTA Gram cut into several K-launches (small gram_launch_kb forces
    5+ launches accumulating into the same partials) agrees with the one-launch
    run and the fp64 reference at the tf32 level."""
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    xd = atucker.DeviceTensor.uniform(list(dims), 29, np.float32)
    ref = gram_np(xd.to_numpy().astype(np.float64), mode)
    try:
        ctx.set_option("gram_launch_kb", 0)
        s1 = atucker.gram(xd, mode)
        ctx.set_option("gram_launch_kb", 64)
        n0 = ctx.launch_count
        sk = atucker.gram(xd, mode)
        n_launch = ctx.launch_count - n0
    finally:
        ctx.set_option("gram_launch_kb", 4096)
    scale = np.abs(ref).max()
    assert n_launch >= 6  # >= 5 Gram launches + the reduction
    assert np.array_equal(sk, sk.T)
    assert np.abs(sk - ref).max() / scale <= 1e-4
    # only the fp32 chain boundaries differ (64 vs 512 K-blocks per chain):
    # measured 5.5e-5 on the diagonal, the tf32 accumulation level
    assert np.abs(sk - s1).max() / scale <= 1e-4


@pytest.mark.parametrize("dims,mode", [
    ((512, 3000), 0), ((768, 2000), 0), ((1280, 900), 0), ((2048, 700), 0),  # nt = 2, 3, 5, 8 tile rows
    ((64, 768, 40), 1), ((32, 1280, 30), 1),                                # K-major panels
])
def test_tc_gram_wide_units(dims, mode):
    """The wide 2-CTA Gram (two tiles of one tile row per unit, A staged once;
    odd rows hand a tile over as its transpose) against the one-tile-per-unit
    kernel and the fp64 reference, at the tf32 level; exactly symmetric."""
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    xd = atucker.DeviceTensor.uniform(list(dims), 41, np.float32)
    ref = gram_np(xd.to_numpy().astype(np.float64), mode)
    try:
        ctx.set_option("gram_wide", 0)
        sn = atucker.gram(xd, mode)
        ctx.set_option("gram_wide", 1)
        sw = atucker.gram(xd, mode)
    finally:
        ctx.set_option("gram_wide", 1)
    scale = np.abs(ref).max()
    assert np.array_equal(sw, sw.T)
    assert np.abs(sw - ref).max() / scale <= 1e-4
    # same tf32 products, same chunking: only the split-K boundaries differ
    assert np.abs(sw - sn).max() / scale <= 1e-4


@pytest.mark.parametrize("dims,mode", [((48, 9000), 0), ((100, 5000), 0), ((128, 3000), 0), ((8, 700), 0),
                                       ((33, 2000), 0), ((8, 48, 301), 1), ((16, 40, 77), 1), ((4, 64, 50, 3), 1)])
def test_tc_gram_small_ring_matches_general(dims, mode):
    """Single-tile Grams (I <= 128; mode 0 or 16-B panels) stage one operand tile per K-block and read it as both A and B
    (option gram_small): the same products, the same fp32 chains and drains as the general ring,
    so the result is bit-identical; and within the tf32 bound of the fp64 Gram."""
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    xd = atucker.DeviceTensor.uniform(list(dims), 5, np.float32)
    out = {}
    try:
        for v in (0, 1):
            ctx.set_option("gram_small", v)
            out[v] = atucker.gram(xd, mode)
    finally:
        ctx.set_option("gram_small", 1)
    np.testing.assert_array_equal(out[0], out[1])
    ref = gram_np(xd.to_numpy().astype(np.float64), mode)
    assert np.abs(out[1] - ref).max() / np.abs(ref).max() <= 4e-3


@pytest.mark.parametrize("dims,r", [
    ((128, 64, 33), 16), ((200, 40, 41), 20), ((2, 7, 5), 1), ((256, 9, 3), 32), ((130, 31), 8),
    ((96, 1000), 24), ((127, 50, 2), 8),
])
def test_fp64_first_mode_ttm(dims, r):
    """fp64 mode-0 TTM (dgemm_ttm: the pipelined DMMA GEMM on the raw tensor, C^T stored): against
    numpy in fp64, odd and even I, R from 1 to 32, J not a multiple of the tile."""
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    xd = atucker.DeviceTensor.uniform(list(dims), 29, np.float64)
    x = xd.to_numpy()
    u = np.random.default_rng(7).standard_normal((r, dims[0]))
    y = atucker.ttm(xd, u, 0, ctx=ctx).to_numpy()
    ref = np.tensordot(u, x, axes=([1], [0]))
    assert y.shape == ref.shape
    np.testing.assert_allclose(y, ref, rtol=0, atol=1e-13 * np.abs(ref).max())
