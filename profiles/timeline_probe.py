"""Probe (not collected): device timeline of the C5 eigensolve (or a whole C5 step) through
torch.profiler's CUPTI activity trace, which records every kernel in the process, the
library's included.  Prints per-kernel device time, the idle gaps between consecutive
kernels, and the span.  Usage: python profiles/timeline_probe.py [eig|step] [out.json]"""
import json
import os
import sys
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import bench  # noqa: E402
from paper_2010_10131_b200 import atucker  # noqa: E402
from paper_2010_10131_b200.selector import Strategy  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "eig"
cfg_name = os.environ.get("ATK_CFG", "c5")  # step mode: which bench config
out = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/timeline.json"
torch.cuda.init()
ctx = atucker.Context.default(0)
for kv in filter(None, os.environ.get("ATK_OPTS", "").split(",")):  # e.g. ATK_OPTS=chol_reg=0
    k, v = kv.split("=")
    ctx.set_option(k, float(v))
cfg = bench.CONFIGS[cfg_name if what == "step" else "c5"]
x = bench.make_input(atucker, cfg, bench.SEEDS[cfg_name if what == "step" else "c5"], ctx)
if what == "eig":
    s0 = atucker.gram(x, 0, ctx=ctx)
    x.free()
    ctx.set_option("eig_assume_psd", 1.0)
    ctx.set_option("chfsi_tol", 1e-10)  # as sthosvd for an fp32 Gram

    def run():
        atucker.sym_eig_top_r(s0, 64, ctx=ctx)
else:
    def run():
        res = atucker.sthosvd(x, cfg["ranks"], Strategy.parse(cfg["strategy"]), ctx=ctx)
        res.decomposition.core.free()
for _ in range(3):
    run()
ctx.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
    ctx.synchronize()
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0, t1 = ev[0]["ts"], max(e["ts"] + e["dur"] for e in ev)
busy = defaultdict(float)
cnt = defaultdict(int)
gaps = []
end = t0
for e in ev:
    name = e["name"].replace("void ", "").replace("atk::(anonymous namespace)::", "").split("(")[0][:60]
    busy[name] += e["dur"]
    cnt[name] += 1
    if e["ts"] > end:
        gaps.append((e["ts"] - end, name))
    end = max(end, e["ts"] + e["dur"])
span = t1 - t0
print(f"span {span:.1f} us, kernels+copies {sum(busy.values()):.1f} us, idle {sum(g for g, _ in gaps):.1f} us "
      f"over {len(gaps)} gaps, {len(ev)} activities")
for k, v in sorted(busy.items(), key=lambda kv: -kv[1])[:30]:
    print(f"{v:10.1f} us {cnt[k]:4d}  {k}")
print("largest gaps (before):")
for g, n in sorted(gaps, reverse=True)[:15]:
    print(f"{g:8.1f} us  {n}")
if len(sys.argv) > 3:  # full listing
    end = t0
    for e in ev:
        n = e["name"].replace("void ", "").replace("atk::(anonymous namespace)::", "").split("(")[0][:60]
        print(f"{e['ts'] - t0:9.1f} gap {e['ts'] - end:7.1f} dur {e['dur']:8.1f}  {n}")
        end = max(end, e["ts"] + e["dur"])
