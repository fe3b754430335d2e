"""Probe (not collected): the n = 192 / 200 dense eigensolve (C1's size) per kernel, CUPTI timeline,
and the trd_kernel phase cycles (ATK_TRD_PROFILE=1)."""
import json
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_10131_b200 import atucker  # noqa: E402

ctx = atucker.Context.default(0)
for n in (160, 192, 200):
    a = np.random.default_rng(n).standard_normal((n, 3 * n))
    s = a @ a.T
    for _ in range(3):
        atucker.sym_eig_top_r(s, 20, ctx=ctx)
    ctx.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        atucker.sym_eig_top_r(s, 20, ctx=ctx)
        ctx.synchronize()
    prof.export_chrome_trace("gpurun_out/trd200.json")
    ev = [e for e in json.load(open("gpurun_out/trd200.json"))["traceEvents"] if e.get("cat") == "kernel"]
    busy = defaultdict(float)
    for e in ev:
        busy[e["name"].split("(")[0][-40:]] += e["dur"]
    print(n, {k: round(v, 1) for k, v in busy.items()}, flush=True)
