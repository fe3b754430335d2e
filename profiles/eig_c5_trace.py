"""Probe (not collected): per-phase GPU times of the C5 mode-0 eigensolve
(ATK_TRACE=events, set before the library loads) on a resident Gram."""
import os
import sys

os.environ["ATK_TRACE"] = "events"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2010_10131_b200 import atucker  # noqa: E402

ctx = atucker.Context.default(0)
cfg = bench.CONFIGS["c5"]
x = bench.make_input(atucker, cfg, bench.SEEDS["c5"], ctx)
# ATK_TRACE stays set: the eigensolver reads it on its first call
s0 = atucker.gram(x, 0, ctx=ctx)
x.free()
ctx.set_option("eig_assume_psd", 1.0)
for _ in range(3):
    atucker.sym_eig_top_r(s0, 64, ctx=ctx)
