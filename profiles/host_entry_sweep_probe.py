"""Probe (not collected): the e2e host-buffer entry (atk_sthosvd_host: chunked upload with the
mode-0 Gram overlapped) against the device entry on the same input, random shapes."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
from paper_2010_10131_b200 import atucker  # noqa: E402
from test_gpu_sweep import _PerMode, _case  # noqa: E402

ctx = atucker.Context.default(0)
bad = 0
n = int(sys.argv[1]) if len(sys.argv) > 1 else 60
for s in range(n):
    dims, ranks, kinds, dtype = _case(s, big=(s % 4 == 0))
    x = np.asfortranarray(np.random.default_rng(s).standard_normal(dims).astype(dtype))
    try:
        a = atucker.sthosvd(x, ranks, _PerMode(kinds), atucker.AlsOptions(seed=2), ctx=ctx)
        b = atucker.sthosvd_host(x, ranks, _PerMode(kinds), atucker.AlsOptions(seed=2), ctx=ctx)
        ga = np.linalg.norm(np.asarray(a.decomposition.core, dtype=np.float64))
        gb = np.linalg.norm(np.asarray(b.decomposition.core, dtype=np.float64))
        tol = 1e-12 if dtype == np.float64 else 1e-5
        if not abs(ga - gb) <= tol * max(ga, 1e-300):
            bad += 1
            print("FAIL", s, dims, ranks, kinds, dtype.__name__, ga, gb, flush=True)
    except Exception as e:  # noqa: BLE001
        bad += 1
        print("ERROR", s, dims, ranks, kinds, dtype.__name__, repr(e)[:200], flush=True)
print(f"done {n}, {bad} bad", flush=True)
