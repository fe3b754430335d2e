"""The B200 roofline selector hook (atk_roofline_selector).

The reference's flop-only cost model (selector.hpp:41-58, heuristic_choice)
routes the big fp32 configs to ALS; on B200 the Gram runs on tensor cores and
ALS is HBM-bound, so the roofline model must keep EIG there.  CPU-only: the
model is host code in libatk_cuda.so and needs no GPU."""
import pytest

from paper_2010_10131_b200.selector import SolverKind, Strategy, heuristic_choice


def _modes(dims, ranks):
    dims = list(dims)
    for n, r in enumerate(ranks):
        j = 1
        for m, d in enumerate(dims):
            if m != n:
                j *= d
        yield n, dims[n], r, j
        dims[n] = r


def test_c5_and_c2_mode1_choose_eig_where_the_flop_model_says_als():
    s = Strategy.roofline("f32")
    picks = [s.decide(n, i, r, j) for n, i, r, j in _modes((2048,) * 3, (64,) * 3)]
    assert picks == [SolverKind.Eig] * 3
    assert [heuristic_choice(i, r, j) for _, i, r, j in _modes((2048,) * 3, (64,) * 3)] == [SolverKind.Als] * 3
    n, i, r, j = next(_modes((1024,) * 3, (32,) * 3))
    assert s.decide(n, i, r, j) == SolverKind.Eig


def test_stage_times_are_rooflines():
    s = Strategy.roofline("f32")
    p = s.roofline_params
    i, r, j = 1024, 32, 1 << 20
    te, ta = s.roofline_times(i, r, j)
    bw, P = p.hbm_gbs * 1e9, p.tf32_tflops * 1e12
    want_e = max(i * i * j / P, 4 * i * j / bw) + p.eig_large_ms * 1e-3 + max(2 * i * r * j / P, 4 * (i + r) * j / bw)
    want_a = (5 * (2 * i + 5 * r) + 2 * r) * 4 * j / bw + 5 * p.als_iter_overhead_ms * 1e-3
    assert te == pytest.approx(want_e, rel=1e-12)
    assert ta == pytest.approx(want_a, rel=1e-12)


def test_fp64_uses_the_fp64_rate_and_overrides_apply():
    f64 = Strategy.roofline("f64")
    f32 = Strategy.roofline("f32")
    assert f64.roofline_times(128, 16, 1 << 21)[0] > f32.roofline_times(128, 16, 1 << 21)[0]
    slow = Strategy.roofline("f32", als_iter_overhead_ms=0.0, eig_large_ms=1e4)
    n, i, r, j = next(_modes((1024,) * 3, (32,) * 3))
    assert slow.decide(n, i, r, j) == SolverKind.Als  # a 10 s eig makes ALS win
    with pytest.raises(Exception):
        Strategy.roofline("f32", bogus=1.0)


def test_parse_and_cpp_header_expose_it():
    from pathlib import Path

    assert Strategy.parse("roofline").kind is Strategy.Kind.Roofline
    hdr = (Path(__file__).resolve().parent.parent / "include" / "atucker_b200.hpp").read_text()
    assert "static Strategy roofline(" in hdr


@pytest.mark.gpu
def test_roofline_hook_drives_sthosvd():
    """The hook plugs into sthosvd like any Strategy (called per mode with the
    shrunk J, sthosvd.hpp:149-166) and its picks show up in the reports."""
    import numpy as np

    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    x = atucker.DeviceTensor.uniform([96, 64, 40], 21, np.float32, ctx=ctx)
    s = Strategy.roofline("f32")
    res = atucker.sthosvd(x, [12, 8, 6], s, ctx=ctx)
    ref = atucker.sthosvd(x, [12, 8, 6], Strategy.fixed_eig(), ctx=ctx)
    dims = [96, 64, 40]
    for n, rep in enumerate(res.reports):
        j = int(np.prod(dims)) // dims[n]
        assert rep.solver_used == s.decide(n, dims[n], [12, 8, 6][n], j)
        dims[n] = [12, 8, 6][n]
    if all(r.solver_used == SolverKind.Eig for r in res.reports):
        np.testing.assert_array_equal(res.decomposition.core.to_numpy(), ref.decomposition.core.to_numpy())


def test_one_pass_als_is_priced_on_mode_0():
    s = Strategy.roofline("f32")
    p = s.roofline_params
    i, r, j = 1024, 32, 1 << 20
    _, two_pass = s.roofline_times(i, r, j)
    _, fused = s.roofline_times(i, r, j, mode=0)
    _, other = s.roofline_times(i, r, j, mode=1)
    assert other == pytest.approx(two_pass, rel=1e-12)
    want = 5 * (p.als_fused_factor * 4 * i * j / (p.hbm_gbs * 1e9) + p.als_fused_overhead_ms * 1e-3)
    assert fused == pytest.approx(want, rel=1e-12) and fused < two_pass
    # not eligible: R > 32 or I not a multiple of 128
    assert s.roofline_times(1000, r, j, mode=0)[1] == pytest.approx(s.roofline_times(1000, r, j)[1], rel=1e-12)
    assert s.roofline_times(i, 48, j, mode=0)[1] == pytest.approx(s.roofline_times(i, 48, j)[1], rel=1e-12)
    # the kernel's per-CTA column bound (als_fused_shape_ok): J above 16384 columns per SM runs
    # the two-pass schedule, so it is priced as such (512 x 2048 x 2048 on mode 0: J = 4M)
    sms = p.num_sms
    assert sms > 0
    j_big = 16384 * sms + 1
    assert s.roofline_times(512, r, j_big, mode=0)[1] == pytest.approx(s.roofline_times(512, r, j_big)[1], rel=1e-12)
    j_ok = 16384 * sms
    assert s.roofline_times(512, r, j_ok, mode=0)[1] < s.roofline_times(512, r, j_ok)[1]
    # and J below one 128-column tile
    assert s.roofline_times(i, r, 100, mode=0)[1] == pytest.approx(s.roofline_times(i, r, 100)[1], rel=1e-12)
