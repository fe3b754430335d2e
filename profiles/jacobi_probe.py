"""One dense PSD Jacobi eig (n = 96) for ncu source-level capture (not a bench)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_10131_b200 import atucker  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96
ctx = atucker.Context.default(0)
ctx.set_option("eig_assume_psd", 1.0)
rng = np.random.default_rng(7)
q = np.linalg.qr(rng.standard_normal((n, n)))[0]
top = 2 * n // 3
lam = np.concatenate([rng.uniform(1, 4, top) * 1e6, rng.uniform(0.9, 1.1, n - top)])
s = (q * lam) @ q.T
p = atucker.sym_eig_top_r(s, top, ctx=ctx)
print("ok", p.values[:3])
