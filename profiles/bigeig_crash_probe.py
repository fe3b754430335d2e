"""Probe (not collected): the dense eigensolver with many wanted vectors (n, r from argv)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_10131_b200 import atucker  # noqa: E402

n, r = int(sys.argv[1]), int(sys.argv[2])
ctx = atucker.Context.default(0)
ctx.set_option("eig_assume_psd", 1.0)
rng = np.random.default_rng(0)
a = rng.standard_normal((n, n + 50))
s = a @ a.T
p = atucker.sym_eig_top_r(s, r, ctx=ctx)
w = np.linalg.eigvalsh(s)[::-1][:r]
print("ok", n, r, np.abs(p.values - w).max() / w[0])
