"""A seeded sweep of st-HOSVD shapes against the oracle (sthosvd.hpp:126-194).

Orders 2-5, dims 1..300 (and 16 fp32 cases up to 2500 / 40M elements), ranks from 1 to the full dim (including ranks equal to
the unfolding's rank bound and modes of size 1), every solver choice per mode
(EIG / ALS / SVD, drawn per case), fp64 and fp32 inputs.  Each case checks the
core norm and the relative reconstruction error against the fp64 oracle, the
orthonormality of every factor, and the core's shape.  Bars: 1e-10 (fp64),
1e-4 (fp32, tf32 tensor-core contractions), north_star's tolerances.
"""
import numpy as np
import pytest

from conftest import orthonormality_defect
from paper_2010_10131_b200.selector import SolverKind, Strategy

pytestmark = pytest.mark.gpu


def _case(seed, big=False):
    rng = np.random.default_rng((5000 if big else 1000) + seed)
    order = int(rng.integers(2, 6)) if not big else int(rng.integers(2, 4))
    budget = (2_000_000 if order <= 3 else 600_000) if not big else 40_000_000
    dims = []
    for n in range(order):
        hi = max(1, min(300 if not big else 2500, int(budget ** (1.0 / order) * 1.8)))
        dims.append(int(rng.integers(1, hi + 1)) if rng.random() < 0.9 else 1)
    while np.prod(dims) > budget:
        k = int(np.argmax(dims))
        dims[k] = max(1, dims[k] // 2)
    # ranks: within each mode's bound as it shrinks (the shrunk unfolding's rank bound for SVD)
    ranks, work = [], list(dims)
    kinds = []
    for n in range(order):
        i = work[n]
        j = int(np.prod(work)) // i
        kind = int(rng.choice([0, 0, 1, 2]))
        hi = min(i, j) if kind == 2 else i
        r = int(rng.integers(1, hi + 1)) if rng.random() < 0.8 else hi
        if kind == 1 and r > min(i, 128):  # keep ALS cases quick
            r = max(1, min(i, 128) // 2)
        if kind == 1 and (2 * r > j or 2 * r > i):
            # GR = rfac rfac^T (r x r) has rank <= J: singular for r > J, where the reference's
            # Cholesky (linalg.hpp:169-177) and this one both stop on a rounding-sized pivot; and
            # near r = I the five iterations invert GR = L^-1 S L^-T with cond(L)^2 cond(S), which
            # amplifies fp64 rounding (any two BLAS orders, Eigen's included) past 1e-10
            kind = 0

        ranks.append(r)
        kinds.append(kind)
        work[n] = r
    dtype = np.float32 if big else (np.float64 if rng.random() < 0.6 else np.float32)
    return dims, ranks, kinds, dtype


class _PerMode(Strategy):
    """Any solver per mode, SVD included (the reference's Manual allows only EIG / ALS,
    sthosvd.hpp:52-55; its hook contract is just decide(mode, i, r, j, params))."""

    def __init__(self, kinds):
        super().__init__(Strategy.Kind.Manual, [SolverKind.Eig] * len(kinds))
        self.kinds = kinds

    def decide(self, mode, i, r, j, params=None):
        return SolverKind(self.kinds[mode])


@pytest.mark.parametrize("seed,big", [(s, False) for s in range(120)] + [(s, True) for s in range(16)])
def test_sthosvd_sweep_vs_oracle(seed, big, oracle):
    """big: fp32 up to 40M elements and dims up to 2500, so the tcgen05 paths run (CTA-pair Gram for
    I >= 512, split-K TTM, the single-tile Gram ring, ALS on the Gram)."""
    from paper_2010_10131_b200 import atucker

    dims, ranks, kinds, dtype = _case(seed, big)
    x = oracle.random_tensor(dims, seed + 7, "normal")
    if dtype == np.float32:
        x = x.astype(np.float32).astype(np.float64)  # the fp32 input, exactly representable
    s = _PerMode(kinds)
    ref = oracle.sthosvd(x, ranks, lambda m, i, r, j: kinds[m], seed=11)
    res = atucker.sthosvd(x.astype(dtype), ranks, s, atucker.AlsOptions(seed=11))
    core = np.asarray(res.decomposition.core, dtype=np.float64)
    assert core.shape == tuple(ranks)
    tol = 1e-10 if dtype == np.float64 else 1e-4
    g, gr = np.linalg.norm(core), np.linalg.norm(ref.core)
    assert abs(g - gr) <= tol * max(gr, 1e-300), (dims, ranks, kinds, dtype, g, gr)
    for f in res.decomposition.factors:
        assert orthonormality_defect(f) <= (1e-10 if dtype == np.float64 else 1e-5)
    e = atucker.relative_error(x, res.decomposition)
    er = oracle.relative_error(x, ref.core, ref.factors)
    # fp32 runs on tf32 tensor-core operands (round-to-nearest, 2^-12 relative): an exactly
    # reconstructible input (er ~ 0) keeps a reconstruction floor of a few 2^-12
    floor = 0.0 if dtype == np.float64 else 4 * 2.0 ** -12
    assert abs(e - er) <= tol * max(1.0, er) + floor, (dims, ranks, kinds, dtype, e, er)


def test_sweep_seed_5339_tiny_fp32_als(oracle):
    """A probe-found case (fp32 22 x 1 x 10 x 1 x 7, ranks 8 x 1 x 7 x 1 x 3, ALS on the last mode,
    whose 5-iteration iterate is first-order sensitive): on tf32 tensor-core operands it missed the
    1e-4 core-norm bar (1.3e-4); tensors below kTcMinElems now take the fp32 CUDA-core path."""
    test_sthosvd_sweep_vs_oracle(5339, False, oracle)
