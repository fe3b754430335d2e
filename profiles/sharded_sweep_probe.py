"""Probe (not collected): the sharded st-HOSVD (host-staged collectives, W ranks sharing the GPU)
against the single-process engine over seeded sweep cases.  Usage:
python profiles/sharded_sweep_probe.py WORLD FIRST LAST"""
import socket
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402


def main():
    import torch.multiprocessing as mp

    from test_gpu_dist import _sweep_worker
    from test_gpu_sweep import _case

    world, a, b = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
    cases = []
    for s in range(a, b):
        dims, ranks, kinds, dtype = _case(s, big=(s % 10 == 0))
        if dims[-1] >= world:
            cases.append((dims, ranks, kinds, dtype))
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    procs = [mpc.Process(target=_sweep_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    bad = 0
    for _ in cases:
        idx, g, gr, de = q.get(timeout=600)
        dims, ranks, kinds, dtype = cases[idx]
        tol = 1e-10 if dtype == np.float64 else 1e-4
        if not (abs(g - gr) <= tol * gr and de <= tol):
            bad += 1
            print("FAIL", cases[idx], g, gr, de, flush=True)
    for p in procs:
        p.join(timeout=120)
    print(f"world {world}: {len(cases)} cases, {bad} failed, exit codes {[p.exitcode for p in procs]}", flush=True)


if __name__ == "__main__":
    main()
