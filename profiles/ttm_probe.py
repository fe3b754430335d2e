"""Probe (not collected): C5 mode-0 TTM alone vs right after the mode-0 Gram (power-cap interplay).
Host wall time around a synchronised call; the device time is within ~50 us of it at these sizes."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2010_10131_b200 import atucker  # noqa: E402

ctx = atucker.Context.default(0)
cfg = bench.CONFIGS["c5"]
x = bench.make_input(atucker, cfg, bench.SEEDS["c5"], ctx)
u = np.linalg.qr(np.random.default_rng(0).standard_normal((2048, 64)))[0].T.copy()


def timed(f):
    ctx.synchronize()
    t0 = time.perf_counter()
    r = f()
    ctx.synchronize()
    return r, (time.perf_counter() - t0) * 1e3


for split in (1, 0):
    ctx.set_option("ttm_split", split)
    for rep in range(4):
        y, dt = timed(lambda: atucker.ttm(x, u, 0, ctx=ctx))
        y.free()
        print(f"split={split} alone rep {rep}: {dt:.3f} ms", flush=True)
    for rep in range(3):
        _, dg = timed(lambda: atucker.gram(x, 0, ctx=ctx))
        y, dt = timed(lambda: atucker.ttm(x, u, 0, ctx=ctx))
        y.free()
        print(f"split={split} after gram ({dg:.1f} ms) rep {rep}: {dt:.3f} ms", flush=True)
