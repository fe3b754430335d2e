"""One C5 st-HOSVD step for profiling under ncu (not a bench number)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2010_10131_b200 import atucker  # noqa: E402
from paper_2010_10131_b200.selector import Strategy  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = bench.CONFIGS[name]
ctx = atucker.Context(0)
import os  # noqa: E402
for kv in filter(None, os.environ.get("ATK_OPTS", "").split(",")):  # e.g. ATK_OPTS=gram_launch_kb=2048
    k, v = kv.split("=")
    ctx.set_option(k, float(v))
x = bench.make_input(atucker, cfg, bench.SEEDS[name], ctx)
for _ in range(steps):
    res = atucker.sthosvd(x, cfg["ranks"], Strategy.parse(cfg["strategy"]), ctx=ctx)
    res.decomposition.core.free()
ctx.synchronize()
print("ok", [round(r.times.total_ms, 2) for r in res.reports])
