"""Probe (not collected): random sym_eig_top_r cases against LAPACK (values 1e-12 of the norm,
orthonormality, residual).  Usage: python profiles/eig_sweep_probe.py N_CASES"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2010_10131_b200 import atucker  # noqa: E402

ctx = atucker.Context.default(0)
n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
bad = 0
for s in range(n_cases):
    rng = np.random.default_rng(9000 + s)
    n = int(rng.choice([1, 2, 3, 5, 17, 48, 80, 112, 113, 128, 150, 200, 201, 256, 400, 700]))
    r = int(rng.integers(1, n + 1)) if rng.random() < 0.5 else min(n, int(rng.integers(1, 65)))
    kind = rng.choice(["gram", "indef", "lowrank", "degen", "flat"])
    q = np.linalg.qr(rng.standard_normal((n, n)))[0]
    if kind == "gram":
        a = rng.standard_normal((n, n + 5))
        sm = a @ a.T
    elif kind == "indef":
        a = rng.standard_normal((n, n))
        sm = 0.5 * (a + a.T)
    elif kind == "lowrank":
        lam = np.concatenate([np.linspace(5, 1, min(n, 10)) * 1e6, rng.uniform(0.9, 1.1, n - min(n, 10))])
        sm = (q * lam) @ q.T
    elif kind == "degen":
        lam = np.repeat(np.linspace(3, 1, (n + 3) // 4), 4)[:n]
        sm = (q * lam) @ q.T
    else:
        lam = 1.0 + 1e-3 * rng.standard_normal(n)
        sm = (q * lam) @ q.T
    sm = 0.5 * (sm + sm.T)
    psd = kind in ("gram", "lowrank", "degen", "flat")
    ctx.set_option("eig_assume_psd", 1.0 if psd else 0.0)
    try:
        p = atucker.sym_eig_top_r(sm, r, ctx=ctx)
        w = np.linalg.eigvalsh(sm)[::-1]
        scale = np.abs(w).max()
        ev = np.abs(p.values - w[:r]).max() / scale
        v = p.vectors
        orth = np.abs(v.T @ v - np.eye(r)).max()
        res = np.abs(sm @ v - v * p.values).max() / scale
        if not (ev <= 1e-12 and orth <= 1e-11 and res <= 1e-10):
            bad += 1
            print("FAIL", s, n, r, kind, f"ev {ev:.2e} orth {orth:.2e} res {res:.2e}", flush=True)
    except Exception as e:  # noqa: BLE001
        bad += 1
        print("ERROR", s, n, r, kind, repr(e)[:200], flush=True)
print(f"done {n_cases}, {bad} bad", flush=True)
