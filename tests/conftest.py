"""Shared test setup.

Markers: `gpu` — needs a B200 (runs under `pytest -m gpu` on the GPU box).
The CPU oracle (oracle/) is the checker; the product package never imports it.
"""
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "4")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA B200 device")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def oracle():
    import oracle as o

    o.load()
    return o


@pytest.fixture(scope="session")
def ctx():
    from paper_2010_10131_b200 import atucker

    return atucker.Context.default(0)


def random_signed(dims, seed, dist="normal"):
    """The reference tests' `random_signed` helpers (mt19937_64 + normal/uniform(-1,1))."""
    import oracle as o

    if dist == "normal":
        return o.random_tensor(dims, seed, "normal")
    u = o.random_tensor(dims, seed, "uniform01")
    return 2.0 * u - 1.0


def principal_angle(a, b) -> float:
    """oracles.hpp:108-114 — largest principal angle between column spaces."""
    qa, _ = np.linalg.qr(a)
    qb, _ = np.linalg.qr(b)
    # sine form ||(I - Qa Qa^T) Qb||_2 resolves angles down to ~1e-16 (arccos of the
    # cosine cannot resolve below ~1e-8)
    s = np.linalg.svd(qb - qa @ (qa.T @ qb), compute_uv=False)
    return float(np.arcsin(min(1.0, s.max())))


def orthonormality_defect(m) -> float:
    """oracles.hpp:117-127."""
    g = m.T @ m
    return float(np.abs(g - np.eye(g.shape[0])).max())
