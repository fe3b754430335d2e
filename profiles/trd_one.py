"""Probe (not collected): one dense eig of a flat Gram of size n (argv[1]), eig_method 3."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_10131_b200 import atucker  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = atucker.Context.default(0)
ctx.set_option("eig_method", 3)
x = np.random.default_rng(0).uniform(-1, 1, (n, 2 * n))
s = x @ x.T
for _ in range(reps):
    p = atucker.sym_eig_top_r(s, 32, ctx=ctx)
print(p.values[:3])
