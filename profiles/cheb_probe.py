"""Flat-spectrum PSD eig at n (default 1024, r 32): exercises the ChFSI filter.

usage: python profiles/cheb_probe.py [n] [r] [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2010_10131_b200 import atucker  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
r = int(sys.argv[2]) if len(sys.argv) > 2 else 32
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
rng = np.random.default_rng(5)
a = rng.random((n, 4 * n))
s = a @ a.T
ctx = atucker.Context.default(0)
ctx.set_option("eig_assume_psd", 1.0)
for _ in range(reps):
    t = time.perf_counter()
    res = atucker.sym_eig_top_r(s, r, ctx=ctx)
    print(f"n={n} r={r}: {1e3 * (time.perf_counter() - t):.2f} ms", flush=True)
w = np.linalg.eigvalsh(s)[::-1][:r]
print("max value err", np.abs(res.values - w).max() / w[0])
