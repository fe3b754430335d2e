"""Probe (not collected): random gram / ttm / sym_eig_top_r shapes against numpy fp64.
Usage: python profiles/kernel_sweep_probe.py N_CASES"""
import sys
import traceback
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_10131_b200 import atucker  # noqa: E402

ctx = atucker.Context.default(0)
n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
bad = 0
for s in range(n_cases):
    rng = np.random.default_rng(7000 + s)
    order = int(rng.integers(1, 5))
    dims = [int(rng.choice([1, 2, 3, 4, 5, 7, 8, 16, 31, 32, 33, 48, 64, 96, 100, 128, 130, 256, 257, 520]))
            for _ in range(order)]
    while np.prod(dims) > 6_000_000:
        k = int(np.argmax(dims))
        dims[k] //= 2
    mode = int(rng.integers(0, order))
    dt = np.float32 if rng.random() < 0.6 else np.float64
    what = rng.choice(["gram", "ttm"])
    try:
        xd = atucker.DeviceTensor.uniform(dims, s, dt, ctx=ctx)
        x = xd.to_numpy().astype(np.float64)
        m = np.moveaxis(x, mode, 0).reshape(dims[mode], -1, order="F")
        tol = 4e-3 if dt == np.float32 else 1e-12
        if what == "gram":
            g = atucker.gram(xd, mode, ctx=ctx)
            ref = m @ m.T
            err = np.abs(g - ref).max() / max(np.abs(ref).max(), 1e-300)
            ok = err <= tol and np.array_equal(g, g.T)
        else:
            r = int(rng.integers(1, min(dims[mode], 140) + 1))
            u = rng.standard_normal((r, dims[mode]))
            y = atucker.ttm(xd, u, mode, ctx=ctx)
            yn = y.to_numpy().astype(np.float64)
            ref = np.moveaxis(np.tensordot(u, x, axes=([1], [mode])), 0, mode)
            err = np.abs(yn - ref).max() / max(np.abs(ref).max(), 1e-300)
            ok = yn.shape == ref.shape and err <= tol
            y.free()
        xd.free()
        if not ok:
            bad += 1
            print("FAIL", s, what, dims, mode, dt.__name__, err, flush=True)
    except Exception as e:  # noqa: BLE001
        bad += 1
        print("ERROR", s, what, dims, mode, dt.__name__, repr(e)[:200], flush=True)
print(f"done {n_cases}, {bad} bad", flush=True)
