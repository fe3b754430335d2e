"""Small invocations of the synchronisation-heavy kernels, for compute-sanitizer
(memcheck / racecheck / synccheck; profiles/sanitize.sh).  Not a bench, not a test.

Cases (argv[1]):
  gram2   fp32 512 x 16 x 16 mode 0: gram_tf32_2cta_kernel (CTA pairs, peer TMA, mbarriers) + gram2_reduce
  gram1   fp32 256 x 8 x 32 modes 0/1: gram_tf32_kernel (1-CTA), ttm_tf32_kernel, ttt
  als     fp32 256 x 64 x 64, ALS mode 0: als_pass_kernel (one-pass ALS) + als_reduce_rows, chol_reg
  chfsi   n = 400 flat PSD Gram: ChFSI (cheb_resident_kernel / cheb_filter_kernel, lanczos_tiles when
          indefinite), CholeskyQR chol_inv, trd_small, bisect / invit / backtr
  trd     n = 120, 190, 193, 200: trd_small_kernel, trd_tile_kernel (193 / 200: the short 7th tile row)
  big     n = 320 dense: the grid-wide Householder reduction (trd_big.cu) + its cluster tail
  svd     fp64 SVD mode on wide and tall unfoldings (svd.cu)
  small   fp32 single-tile Gram ring (mode 0 and 16-B panels), gram_tc.cu
  f64     fp64 SYRK Gram and DMMA-GEMM TTM (dgemm.cu), first and last modes
  alsgram ALS on the Gram (driver.cu), fp32 mode 0
  bigeig  dense eigensolver above n = 2048 (the <8, 32> grid instance)
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_10131_b200 import atucker  # noqa: E402
from paper_2010_10131_b200.selector import SolverKind, Strategy  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "gram2"
ctx = atucker.Context.default(0)
rng = np.random.default_rng(1)


def sym(n, kind):
    q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    lam = np.sort(1.0 + 0.06 * rng.standard_normal(n))[::-1] if kind == "flat" else np.linspace(n, 1, n)
    return (q * lam) @ q.T


if case == "gram2":
    x = atucker.DeviceTensor.uniform([512, 16, 16], 3, np.float32, ctx=ctx)
    res = atucker.sthosvd(x, [16, 8, 8], Strategy.fixed_eig(), ctx=ctx)
elif case == "gram1":
    x = atucker.DeviceTensor.uniform([256, 8, 32], 3, np.float32, ctx=ctx)
    res = atucker.sthosvd(x, [32, 4, 8], Strategy.fixed_eig(), ctx=ctx)
elif case == "als":
    x = atucker.DeviceTensor.uniform([256, 64, 64], 5, np.float32, ctx=ctx)
    res = atucker.sthosvd(x, [16, 16, 16], Strategy.manual([SolverKind.Als, SolverKind.Eig, SolverKind.Eig]),
                          atucker.AlsOptions(num_iters=2, seed=3), ctx=ctx)
elif case == "chfsi":  # (also the persistent scratch and the early result enqueue)
    ctx.set_option("eig_assume_psd", 1.0)
    ctx.set_option("eig_method", 1)
    p = atucker.sym_eig_top_r(sym(400, "flat"), 24, ctx=ctx)
    ctx.set_option("eig_assume_psd", 0.0)
    p = atucker.sym_eig_top_r(sym(400, "lin") - 100.0 * np.eye(400), 24, ctx=ctx)
    ctx.set_option("eig_method", -1)
elif case == "trd":
    for n in (120, 190, 193, 200):  # 193 / 200: the tile reduction's short 7th tile row
        p = atucker.sym_eig_top_r(sym(n, "lin"), 16, ctx=ctx)
elif case == "big":
    ctx.set_option("eig_method", 3)
    p = atucker.sym_eig_top_r(sym(320, "flat"), 20, ctx=ctx)
    ctx.set_option("eig_method", -1)
elif case == "svd":
    for dims, mode, r in (([24, 10, 12], 0, 8), ([40, 3, 4], 0, 6)):
        y = np.asfortranarray(rng.standard_normal(dims))
        atucker.svd_mode_solver(y, mode, r, ctx=ctx)
elif case == "small":
    for dims, mode in (([48, 2000], 0), ([8, 48, 301], 1), ([100, 700], 0)):
        x = atucker.DeviceTensor.uniform(dims, 3, np.float32, ctx=ctx)
        atucker.gram(x, mode, ctx=ctx)
elif case == "f64":
    x = np.asfortranarray(rng.standard_normal((128, 40, 30)))
    res = atucker.sthosvd(x, [16, 8, 6], Strategy.fixed_eig(), ctx=ctx)
elif case == "alsgram":
    x = atucker.DeviceTensor.uniform([512, 64, 64], 5, np.float32, ctx=ctx)
    atucker.als_mode_solver(x, 0, 16, atucker.AlsOptions(num_iters=2, seed=3), ctx=ctx)
elif case == "bigeig":
    ctx.set_option("eig_method", 3)
    a = rng.standard_normal((2100, 2100))
    p = atucker.sym_eig_top_r(0.5 * (a + a.T), 8, ctx=ctx)
    ctx.set_option("eig_method", -1)
else:
    raise SystemExit(f"unknown case {case}")
ctx.synchronize()
print("ok", case)
