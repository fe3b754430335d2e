"""Probe (not collected): special inputs through sthosvd vs the oracle (zeros, constants, a single
element, rank-1, huge / tiny scales) for every solver; reports errors instead of crashing."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
sys.path.insert(0, str(ROOT / "tests"))
import oracle as o  # noqa: E402
from paper_2010_10131_b200 import atucker  # noqa: E402
from test_gpu_sweep import _PerMode  # noqa: E402

o.load()
cases = {
    "zeros": np.zeros((20, 30, 40)),
    "const": np.full((20, 30, 40), 3.0),
    "one": np.full((1, 1, 1), 2.0),
    "rank1": np.einsum("i,j,k->ijk", np.arange(1, 21.0), np.ones(30), np.linspace(1, 2, 40)),
    "huge": np.random.default_rng(0).standard_normal((20, 30, 40)) * 1e140,
    "tiny": np.random.default_rng(1).standard_normal((20, 30, 40)) * 1e-140,
}
for name, x in cases.items():
    for kinds in ([0, 0, 0], [1, 1, 1], [2, 2, 2], [0, 1, 2]):
        ranks = [min(3, d) for d in x.shape]
        for dt in (np.float64, np.float32):
            if dt == np.float32 and name in ("huge", "tiny"):
                continue
            xx = np.asfortranarray(x.astype(dt))
            msg = ""
            try:
                ref = o.sthosvd(xx.astype(np.float64), ranks, lambda m, i, r, j: kinds[m], seed=1)
                gr = np.linalg.norm(ref.core)
            except Exception as e:  # noqa: BLE001
                ref, gr, msg = None, None, f"oracle {type(e).__name__}"
            try:
                res = atucker.sthosvd(xx, ranks, _PerMode(kinds), atucker.AlsOptions(seed=1))
                g = np.linalg.norm(np.asarray(res.decomposition.core, dtype=np.float64))
                ok = gr is not None and (abs(g - gr) <= (1e-10 if dt == np.float64 else 1e-4) * max(gr, 1e-300) or gr == g)
                print(f"{name:6s} {kinds} {dt.__name__}: engine |G| {g:.6e} oracle {gr} {'OK' if ok else 'DIFF'} {msg}",
                      flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"{name:6s} {kinds} {dt.__name__}: engine {type(e).__name__}: {str(e)[:80]} | {msg}", flush=True)
