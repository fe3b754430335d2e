"""Probe (not collected): the 2-CTA Gram with 4096 vs 1024 K-blocks per unit and launch must be
bit-identical (the fp32 drains every 512 K-blocks fall on the same K boundaries)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_10131_b200 import atucker  # noqa: E402

for dims, mode in (([2048, 2048, 512], 0), ([1024, 4096, 300], 0), ([64, 2048, 2048], 1), ([2048, 1000, 700], 1)):
    g = {}
    for kb in (4096, 1024, 2048):
        ctx = atucker.Context(0)
        ctx.set_option("gram_launch_kb", kb)
        x = atucker.DeviceTensor.uniform(dims, 17, np.float32, ctx=ctx)
        g[kb] = atucker.gram(x, mode, ctx=ctx)
        x.free()
    same = all(np.array_equal(g[4096], g[k]) for k in (1024, 2048))
    print(dims, mode, "bit-identical" if same else f"DIFFER max {np.abs(g[4096] - g[1024]).max():.3e}", flush=True)
