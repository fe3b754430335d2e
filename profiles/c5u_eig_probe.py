"""Probe (not collected): the C5 stress Grams (uniform 2048^3 fp32, seed 5),
modes 0 and 1, through the default eig dispatch (ChFSI -> dense hand-over) and
the dense solver alone, with ATK_TRACE on.  Saves the mode-0 Gram to
gpurun_out/c5u_gram0.npy for spectrum analysis on the CPU."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_10131_b200 import atucker  # noqa: E402

ctx = atucker.Context.default(0)
x = atucker.DeviceTensor.uniform([2048, 2048, 2048], 5, np.float32, ctx=ctx)
s0 = atucker.gram(x, 0, ctx=ctx)
os.makedirs("gpurun_out", exist_ok=True)
np.save("gpurun_out/c5u_gram0.npy", s0)
ctx.set_option("eig_assume_psd", 1.0)
for method in (-1, 3, 1):
    ctx.set_option("eig_method", method)
    for rep in range(2):
        t0 = time.perf_counter()
        try:
            p = atucker.sym_eig_top_r(s0, 64, ctx=ctx)
            ok = f"theta_1 {p.values[0]:.6e} theta_64 {p.values[-1]:.6e}"
        except Exception as e:  # noqa: BLE001
            ok = f"error {e}"
        print(f"method {method} rep {rep}: host {1e3 * (time.perf_counter() - t0):.1f} ms {ok}", flush=True)
