"""Probe (not collected): device timeline (CUPTI via torch.profiler) of the exact dense
eigensolver at n = 2048 on a flat-spectrum Gram (the C5u stress case), eig_method 3."""
import json
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2010_10131_b200 import atucker  # noqa: E402

torch.cuda.init()
ctx = atucker.Context.default(0)
ctx.set_option("eig_assume_psd", 1.0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
method = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rng = np.random.default_rng(0)
x = rng.uniform(0, 1, (n, 2 * n))
s = x @ x.T
ctx.set_option("eig_method", method)
for _ in range(2):
    atucker.sym_eig_top_r(s, 64, ctx=ctx)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    atucker.sym_eig_top_r(s, 64, ctx=ctx)
out = "gpurun_out/bigeig_tl.json"
prof.export_chrome_trace(out)
ev = [e for e in json.load(open(out))["traceEvents"] if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
busy, cnt = defaultdict(float), defaultdict(int)
for e in ev:
    k = e["name"].replace("void ", "").replace("atk::(anonymous namespace)::", "").split("(")[0][:60]
    busy[k] += e["dur"]
    cnt[k] += 1
print(f"n={n} method={method}: span {max(e['ts'] + e['dur'] for e in ev) - ev[0]['ts']:.0f} us")
for k, v in sorted(busy.items(), key=lambda kv: -kv[1])[:15]:
    print(f"{v:10.1f} us {cnt[k]:4d}  {k}")
