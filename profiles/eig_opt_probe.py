"""One dense eig under option combinations (ATK_TRACE=1 for the ChFSI trace).

usage: python profiles/eig_opt_probe.py N [psd] [method]
Runs lanczos_tiles x cheb_fused in {1, 0} x {1, 2} and reports errors vs LAPACK.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

from paper_2010_10131_b200 import atucker

n = int(sys.argv[1])
psd = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
method = int(sys.argv[3]) if len(sys.argv) > 3 else 0
rng = np.random.default_rng(n)
a = rng.standard_normal((n, n + 7))
s = a @ a.T
r = int(sys.argv[4]) if len(sys.argv) > 4 else max(1, n // 2)
w = np.linalg.eigvalsh(s)[::-1][:r]
for lt in (1, 0):
    for cf in (1, 2):
        ctx = atucker.Context.default(0)
        ctx.set_option("eig_assume_psd", psd)
        ctx.set_option("eig_method", method)
        ctx.set_option("lanczos_tiles", lt)
        ctx.set_option("cheb_fused", cf)
        try:
            res = atucker.sym_eig_top_r(s, r, ctx=ctx)
            print(f"lanczos_tiles={lt} cheb_fused={cf}: max value err {np.abs(res.values - w).max() / w[0]:.3e}",
                  flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"lanczos_tiles={lt} cheb_fused={cf}: {type(e).__name__}: {e}", flush=True)
