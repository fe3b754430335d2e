"""Memory discipline on the device (the reference's AllocTracker checks).

Restated from:
* acceptance.cpp:428-458, criterion 12: an EIG or ALS st-HOSVD holds at most one buffer of the
  input's size. The reference holds exactly one, its `work = x` copy. The engine never copies the
  input, so it holds none.
* test_kernels.cpp:140-148: a TTM allocates only its output. There is exactly one allocation, no
  buffer of the input's size, and nothing is live once the result is freed.

The reference's explicit-SVD path materialises an unfolding (its peak is at least 2: the work copy
plus the unfolding). The engine's SVD mode works on the explicit unfolding too (svd.cu) but keeps
no work copy, so its check is "at least one, at most two".
"""
import numpy as np
import pytest

from paper_2010_10131_b200.selector import Strategy

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("strategy", ["eig", "als", "svd"])
def test_criterion12_memory_discipline(strategy):
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    x = atucker.DeviceTensor.uniform([24, 20, 16], 1012, np.float64, ctx=ctx)
    st = {"eig": Strategy.fixed_eig(), "als": Strategy.fixed_als(), "svd": Strategy.fixed_svd()}[strategy]
    with atucker.AllocScope(24 * 20 * 16) as scope:
        res = atucker.sthosvd(x, [8, 8, 8], st, atucker.AlsOptions(seed=3), ctx=ctx)
        stats = scope.stats()
    assert stats["alloc_count"] > 0  # the shrunk tensors and the core are tracked
    if strategy == "svd":
        # acceptance.cpp:450-455: the explicit path materialises an unfolding
        assert 1 <= stats["peak_watched"] <= 2, stats
    else:
        assert stats["peak_watched"] == 0, stats  # no copy of the input at all
    res.decomposition.core.free()


def test_ttm_allocates_only_its_output():
    from paper_2010_10131_b200 import atucker

    ctx = atucker.Context.default(0)
    x = atucker.DeviceTensor.uniform([6, 7, 8], 11, np.float64, ctx=ctx)
    u = np.random.default_rng(13).standard_normal((3, 7))
    with atucker.AllocScope(6 * 7 * 8) as scope:
        y = atucker.ttm(x, u, 1, ctx=ctx)
        y.free()
        stats = scope.stats()
    assert stats["alloc_count"] == 1
    assert stats["peak_watched"] == 0
    assert stats["live_elems"] == 0
