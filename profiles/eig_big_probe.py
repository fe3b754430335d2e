"""Probe (not collected): dense (trd_big) vs ChFSI on flat / gapped Grams, ATK_TRACE on."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("ATK_TRACE", "1")
from paper_2010_10131_b200 import atucker  # noqa: E402

ctx = atucker.Context.default(0)
ctx.set_option("eig_assume_psd", 1.0)
rng = np.random.default_rng(0)
for n, r in [(256, 20), (512, 32), (1024, 32), (1024, 64), (2048, 64)]:
    x = rng.uniform(-1, 1, (n, 4 * n))
    s = x @ x.T
    w = np.linalg.eigvalsh(s)[::-1][:r]
    for method in (3, -1):
        ctx.set_option("eig_method", method)
        for rep in range(2):
            t0 = time.perf_counter()
            p = atucker.sym_eig_top_r(s, r, ctx=ctx)
            dt = time.perf_counter() - t0
        print(f"n={n} r={r} method={method}: host {dt*1e3:.1f} ms, max rel eigval err "
              f"{np.abs(p.values - w).max() / w.max():.2e}", flush=True)
