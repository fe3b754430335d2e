"""World-size-2 CPU tests of the multi-GPU st-HOSVD algorithm (gloo).

The engine's sharded schedule (csrc/dist.cu + driver.cu): shard the last
mode, per mode n < N-1 compute the local Gram, allreduce it, solve the
replicated eig, TTM locally; before the last mode all-gather the (small)
shrunk tensor and finish replicated.  ALS modes allreduce YR and GR per
iteration (driver.cu als_iterate).  Here the same schedule runs with the
CPU oracle as the per-shard compute and torch.distributed gloo as the
collective, and must reproduce the single-process st-HOSVD."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2010_10131_b200.dist import shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _allreduce(a):
    t = torch.from_numpy(np.ascontiguousarray(a))
    dist.all_reduce(t)
    return np.asfortranarray(t.numpy())


def _sharded_als(o, y, n, r, seed, sharded, iters=5):
    """driver.cu als_iterate / als_mode under a communicator: W, rfac and the
    shrunk tensor stay local; YR (I x r) and GR (r x r) are sums over J and are
    allreduced once per iteration; L and every r x r solve are replicated."""
    L = o.als_initial_guess(y.shape[n], r, seed, n)
    eye = np.eye(r, order="F")
    for _ in range(iters):
        w = o.ttm(y, L.T, n)
        rfac = o.ttm(w, o.spd_solve(o.gemm(L, L, trans_a=True), eye), n)
        yr, gr = o.ttt_mode(y, rfac, n), o.ttt_mode(rfac, rfac, n)
        if sharded:
            yr, gr = _allreduce(yr), _allreduce(gr)
        L = o.gemm(yr, o.spd_solve(gr, eye))
    q, rr = o.thin_qr(L)
    return q, o.ttm(rfac, rr, n)


def _sharded_sthosvd(o, x_local, ranks, kinds=None, seed=0):
    order = x_local.ndim
    kinds = kinds or [0] * order
    work = x_local
    factors = []
    for n in range(order):
        if n == order - 1:  # gather the shard mode
            parts = [None] * dist.get_world_size()
            dist.all_gather_object(parts, work)
            work = np.asfortranarray(np.concatenate(parts, axis=order - 1))
        if kinds[n] == 1:
            f, work = _sharded_als(o, work, n, ranks[n], seed, n < order - 1)
            factors.append(f)
            continue
        s = o.gram(work, n)
        if n < order - 1:
            s = _allreduce(s)
        p = o.sym_eig_top_r(s, ranks[n])
        factors.append(p.vectors)
        work = o.ttm(work, p.vectors.T, n)
    return work, factors


def _worker(rank, world, port, dims, ranks, out, kinds=None):
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle as o

    x = o.random_tensor(dims, 7, "normal")
    lo, hi = shard_range(dims[-1], rank, world)
    core, factors = _sharded_sthosvd(o, np.asfortranarray(x[..., lo:hi]), ranks, kinds, seed=11)
    if rank == 0:
        ref = o.sthosvd(x, ranks, (lambda m, i, r, j: kinds[m]) if kinds else None, seed=11)
        out.put((np.linalg.norm(core), np.linalg.norm(ref.core),
                 max(np.abs(a - b).max() for a, b in zip(factors, ref.factors))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dims,ranks,kinds", [((12, 10, 9), (4, 3, 3), None),
                                              ((8, 7, 6, 5), (3, 3, 2, 2), None),
                                              ((12, 10, 9), (4, 3, 3), [1, 0, 1]),
                                              ((8, 7, 6, 5), (3, 3, 2, 2), [0, 1, 1, 0])])
def test_sharded_schedule_matches_single_process(dims, ranks, kinds):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dims, ranks, q, kinds)) for r in range(2)]
    for p in procs:
        p.start()
    g, gr, fdiff = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert abs(g - gr) / gr <= 1e-12
    assert fdiff <= (1e-8 if kinds else 1e-10)  # deterministic eig => same factors (sign rule) on every rank


def test_shard_range_partitions():
    for n in (1, 7, 2048):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
