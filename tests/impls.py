"""Two implementations behind one test-facing interface.

`OracleImpl` is the CPU restatement (the checker); `EngineImpl` is the
product (libatk_cuda.so through the C ABI).  The reference's own test suites
(tests/test_*.cpp, acceptance.cpp) are restated once against this interface
and run on both: on CPU they pin the oracle, on the GPU (`-m gpu`) they test
the engine.  Parity tests then compare the two directly.
"""
from __future__ import annotations

import numpy as np


class OracleImpl:
    name = "oracle"

    def __init__(self):
        import oracle as o

        self.o = o
        o.load()

    def frobenius_norm(self, x):
        return self.o.frobenius_norm(x)

    def gram(self, x, n):
        return self.o.gram(x, n)

    def ttm(self, x, u, n):
        return self.o.ttm(x, u, n)

    def ttt(self, x, y, n):
        return self.o.ttt_mode(x, y, n)

    def eig(self, s, r):
        p = self.o.sym_eig_top_r(s, r)
        return p.values, p.vectors

    def qr(self, a):
        return self.o.thin_qr(a)

    def spd_solve(self, a, b):
        return self.o.spd_solve(a, b)

    def eig_mode(self, y, n, r):
        m = self.o.eig_mode_solver(y, n, r)
        return m.factor, m.shrunk

    def svd_mode(self, y, n, r):
        m = self.o.svd_mode_solver(y, n, r)
        return m.factor, m.shrunk

    def als_mode(self, y, n, r, num_iters=5, rel_tol=0.0, seed=0):
        m = self.o.als_mode_solver(y, n, r, num_iters, rel_tol, seed)
        return m.factor, m.shrunk, m.iterations_run

    def als_iterate(self, y, n, l0, num_iters=5, rel_tol=0.0):
        l, rfac, it, _ = self.o.als_iterate(y, n, l0, num_iters, rel_tol)
        return l, rfac, it

    def sthosvd(self, x, ranks, strategy=None, num_iters=5, rel_tol=0.0, seed=0):
        from paper_2010_10131_b200.selector import CostModelParams, Strategy

        strategy = strategy or Strategy.fixed_eig()
        if strategy.kind is Strategy.Kind.Manual and len(strategy.choices) != np.ndim(x):
            from paper_2010_10131_b200.errors import Error  # sthosvd.hpp:138-140

            raise Error(f"manual strategy must choose a solver for each of the {np.ndim(x)} modes")
        params = CostModelParams(num_iters)
        res = self.o.sthosvd(x, ranks, lambda m, i, r, j: int(strategy.decide(m, i, r, j, params)),
                             num_iters, rel_tol, seed)
        return res.core, res.factors, [int(v) for v in res.reports[:, 0]]

    def reconstruct(self, core, factors, dims):
        return self.o.reconstruct(core, factors, dims)

    def relative_error(self, x, core, factors):
        return self.o.relative_error(x, core, factors)

    def reset_counters(self):
        self.o.reset_counters()

    def counters(self):
        return self.o.gemm_calls(), self.o.gemm_flops()


class EngineImpl:
    name = "engine"

    def __init__(self):
        from paper_2010_10131_b200 import atucker

        self.a = atucker
        self.ctx = atucker.Context.default(0)

    def frobenius_norm(self, x):
        return self.a.frobenius_norm(x)

    def gram(self, x, n):
        return self.a.gram(x, n)

    def ttm(self, x, u, n):
        return self.a.ttm(x, u, n)

    def ttt(self, x, y, n):
        return self.a.ttt_mode(x, y, n)

    def eig(self, s, r):
        p = self.a.sym_eig_top_r(s, r)
        return p.values, p.vectors

    def qr(self, a):
        p = self.a.thin_qr(a)
        return p.q, p.r

    def spd_solve(self, a, b):
        b = np.asarray(b, dtype=np.float64)
        if b.ndim == 1:
            b = b.reshape(-1, 1)
        return self.a.spd_solve(a, b)

    def eig_mode(self, y, n, r):
        m = self.a.eig_mode_solver(y, n, r)
        return m.factor, m.shrunk

    def svd_mode(self, y, n, r):
        m = self.a.svd_mode_solver(y, n, r)
        return m.factor, m.shrunk

    def als_mode(self, y, n, r, num_iters=5, rel_tol=0.0, seed=0):
        m = self.a.als_mode_solver(y, n, r, self.a.AlsOptions(num_iters, rel_tol, seed))
        return m.factor, m.shrunk, m.iterations_run

    def als_iterate(self, y, n, l0, num_iters=5, rel_tol=0.0):
        res = self.a.als_iterate(y, n, l0, self.a.AlsOptions(num_iters, rel_tol, 0))
        return res.l, res.rfac, res.iterations_run

    def sthosvd(self, x, ranks, strategy=None, num_iters=5, rel_tol=0.0, seed=0):
        res = self.a.sthosvd(x, ranks, strategy, self.a.AlsOptions(num_iters, rel_tol, seed))
        d = res.decomposition
        return d.core, d.factors, [int(r.solver_used) for r in res.reports]

    def reconstruct(self, core, factors, dims):
        return self.a.reconstruct(self.a.TuckerDecomposition(core, factors, tuple(dims)))

    def relative_error(self, x, core, factors):
        return self.a.relative_error(x, self.a.TuckerDecomposition(core, factors, tuple(np.shape(x))))

    def reset_counters(self):
        self.a.reset_gemm_counters()

    def counters(self):
        return self.a.gemm_calls(), self.a.gemm_flops()


_CACHE: dict = {}


def get(name: str):
    if name not in _CACHE:
        _CACHE[name] = OracleImpl() if name == "oracle" else EngineImpl()
    return _CACHE[name]
