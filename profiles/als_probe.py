"""ALS mode timing on C2 (1024^3 f32, r = 32, mode 0), repeated: run with ATK_TRACE=1."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_10131_b200 import atucker  # noqa: E402

import os  # noqa: E402

ctx = atucker.Context(0)
if "ALS_HEAD" in os.environ:  # phase-1 K-blocks ahead of phase 2 (option als_head; -1 = no overlap)
    ctx.set_option("als_head", int(os.environ["ALS_HEAD"]))
x = atucker.DeviceTensor.uniform([1024, 1024, 1024], 2, np.float32, ctx=ctx)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    ctx.synchronize()
    t0 = time.perf_counter()
    res = atucker.als_mode_solver(x, 0, 32, ctx=ctx)
    ctx.synchronize()
    print(f"rep {rep}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
