"""Probe (not collected): the C5 (low-rank) mode-0 Gram's eigensolve, timed
in isolation (device events around repeated sym_eig_top_r calls on a resident
Gram), default vs ATK_INVIT_SEQ=1, then one ATK_TRACE=events run."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2010_10131_b200 import atucker  # noqa: E402

ctx = atucker.Context.default(0)
cfg = bench.CONFIGS["c5"]
x = bench.make_input(atucker, cfg, bench.SEEDS["c5"], ctx)
s0 = atucker.gram(x, 0, ctx=ctx)
x.free()
ctx.set_option("eig_assume_psd", 1.0)
for env in ("", "1"):
    if env:
        os.environ["ATK_INVIT_SEQ"] = env
    else:
        os.environ.pop("ATK_INVIT_SEQ", None)
    for _ in range(2):
        atucker.sym_eig_top_r(s0, 64, ctx=ctx)
    ctx.synchronize()
    t = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        atucker.sym_eig_top_r(s0, 64, ctx=ctx)
        b.record()
        torch.cuda.synchronize()
        t.append(a.elapsed_time(b))
    print(f"ATK_INVIT_SEQ={env or 0}: eig n=2048 r=64 median {np.median(t):.3f} ms (host-inclusive, incl. H2D of S)",
          flush=True)
os.environ.pop("ATK_INVIT_SEQ", None)
os.environ["ATK_TRACE"] = "events"
atucker.sym_eig_top_r(s0, 64, ctx=ctx)
