"""World-size-2 CPU tests of the multi-GPU st-HOSVD algorithm (gloo).

The engine's sharded schedule (csrc/dist.cu + driver.cu): shard the last
mode, per mode n < N-1 compute the local Gram, allreduce it, solve the
replicated eig, TTM locally; before the last mode all-gather the (small)
shrunk tensor and finish replicated.  Here the same schedule runs with the
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


def _sharded_sthosvd(o, x_local, ranks):
    order = x_local.ndim
    work = x_local
    factors = []
    for n in range(order):
        if n == order - 1:  # gather the shard mode
            parts = [None] * dist.get_world_size()
            dist.all_gather_object(parts, work)
            work = np.asfortranarray(np.concatenate(parts, axis=order - 1))
        s = o.gram(work, n)
        if n < order - 1:
            t = torch.from_numpy(np.ascontiguousarray(s))
            dist.all_reduce(t)
            s = np.asfortranarray(t.numpy())
        p = o.sym_eig_top_r(s, ranks[n])
        factors.append(p.vectors)
        work = o.ttm(work, p.vectors.T, n)
    return work, factors


def _worker(rank, world, port, dims, ranks, out):
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
    core, factors = _sharded_sthosvd(o, np.asfortranarray(x[..., lo:hi]), ranks)
    if rank == 0:
        ref = o.sthosvd(x, ranks)
        out.put((np.linalg.norm(core), np.linalg.norm(ref.core),
                 max(np.abs(a - b).max() for a, b in zip(factors, ref.factors))))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dims,ranks", [((12, 10, 9), (4, 3, 3)), ((8, 7, 6, 5), (3, 3, 2, 2))])
def test_sharded_schedule_matches_single_process(dims, ranks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, dims, ranks, q)) for r in range(2)]
    for p in procs:
        p.start()
    g, gr, fdiff = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert abs(g - gr) / gr <= 1e-12
    assert fdiff <= 1e-10  # deterministic eig => same factors (sign rule) on every rank


def test_shard_range_partitions():
    for n in (1, 7, 2048):
        for w in (1, 2, 3, 8):
            spans = [shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
