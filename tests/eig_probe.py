"""Ad-hoc probe (not collected by pytest): eig stage trace on a C5-like Gram."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_10131_b200 import atucker  # noqa: E402

n, r = int(sys.argv[1]) if len(sys.argv) > 1 else 2048, 64
rng = np.random.default_rng(0)
atucker.Context.default(0).set_option("eig_assume_psd", 1.0)  # as the driver: Grams are PSD
for kind in ["lowrank", "flat"]:
    if kind == "lowrank":
        q = np.linalg.qr(rng.standard_normal((n, n)))[0]
        lam = np.concatenate([np.sort(rng.uniform(1, 4, r))[::-1] * 1e6, rng.uniform(0.9, 1.1, n - r)])
    else:
        q = np.linalg.qr(rng.standard_normal((n, n)))[0]
        lam = np.sort(1.0 + 0.06 * rng.standard_normal(n))[::-1]
    s = (q * lam) @ q.T
    for rep in range(2):
        t0 = time.perf_counter()
        p = atucker.sym_eig_top_r(s, r)
        dt = time.perf_counter() - t0
    ref = np.sort(lam)[::-1][:r]
    print(f"{kind}: {dt*1e3:.1f} ms, max rel eigval err {np.abs(p.values - ref).max() / ref.max():.2e}", flush=True)

ctx = atucker.Context.default(0)
for psd in (0.0, 1.0):
  ctx.set_option("eig_assume_psd", psd)
  for m in (48, 96, 112, 128, 152):
    a = rng.standard_normal((m, m + 7))
    s = a @ a.T
    for rep in range(3):
        t0 = time.perf_counter()
        p = atucker.sym_eig_top_r(s, m // 2)
        dt = time.perf_counter() - t0
    w = np.linalg.eigvalsh(s)[::-1][: m // 2]
    print(f"dense jacobi psd={psd} n={m}: {dt*1e3:.3f} ms, rel err {np.abs(p.values - w).max() / w.max():.2e}", flush=True)
