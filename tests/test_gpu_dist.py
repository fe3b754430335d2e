"""The multi-GPU code path (csrc/dist.cu) on the one GPU available.

Every GPU run this round has a single GPU, so N > 1 cannot execute here. A world-size-1 NCCL
communicator still drives the whole sharded schedule through the real NCCL calls: the
dlopen'ed libnccl, ncclCommInitRank, the per-mode fp64 Gram allreduce, and the grouped-broadcast
all-gather before the last mode. Its results must be bit-identical to the communicator-free run,
because a 1-rank sum is a copy. The N > 1 planning logic is covered by tests/test_dist_gloo.py.
"""
import numpy as np
import pytest

from paper_2010_10131_b200.selector import Strategy

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_world1_nccl_matches_single(dtype):
    from paper_2010_10131_b200 import atucker

    dims, ranks = [96, 40, 33], [12, 8, 5]
    plain = atucker.Context(0)
    xd = atucker.DeviceTensor.uniform(dims, 17, dtype, ctx=plain)
    ref = atucker.sthosvd(xd, ranks, Strategy.fixed_eig(), ctx=plain)

    dist = atucker.Context(0)
    dist.comm_init(atucker.Context.nccl_unique_id(), 0, 1)
    xh = xd.to_numpy()
    xd2 = atucker.DeviceTensor.from_numpy(xh, ctx=dist)
    res = atucker.sthosvd(xd2, ranks, Strategy.fixed_eig(), ctx=dist, global_dims=dims)

    g0 = ref.decomposition.core.to_numpy()
    g1 = res.decomposition.core.to_numpy()
    np.testing.assert_array_equal(g0, g1)
    for a, b in zip(ref.decomposition.factors, res.decomposition.factors):
        np.testing.assert_array_equal(a, b)


def _host_comm_worker(rank, world, port, dims, ranks, kinds, dtype, out):
    import os
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2010_10131_b200 import atucker
    from paper_2010_10131_b200.dist import init_host_comm_from_torch, shard_range
    from paper_2010_10131_b200.selector import SolverKind, Strategy

    rng = np.random.default_rng(5)
    x = np.asfortranarray(rng.standard_normal(dims).astype(dtype))
    strat = Strategy.manual([SolverKind(k) for k in kinds])
    opts = atucker.AlsOptions(seed=9)
    ctx = atucker.Context(0)
    init_host_comm_from_torch(ctx)
    lo, hi = shard_range(dims[-1], rank, world)
    xl = atucker.DeviceTensor.from_numpy(np.asfortranarray(x[..., lo:hi]), ctx=ctx)
    res = atucker.sthosvd(xl, ranks, strat, opts, ctx=ctx, global_dims=dims)
    core = res.decomposition.core.to_numpy().astype(np.float64)
    facs = res.decomposition.factors
    comm_ms = sum(r.times.comm_ms for r in res.reports)
    if rank == 0:
        plain = atucker.Context(0)
        plain.set_option("als_gram", 0)  # the sharded run iterates over Y (the Gram route is single-GPU)
        ref = atucker.sthosvd(atucker.DeviceTensor.from_numpy(x, ctx=plain), ranks, strat, opts, ctx=plain)
        g, gr = np.linalg.norm(core), np.linalg.norm(ref.decomposition.core.to_numpy().astype(np.float64))
        fd = max(np.abs(a - b).max() for a, b in zip(facs, ref.decomposition.factors))
        out.put((g, gr, fd, comm_ms))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dims,ranks,kinds,dtype,tol", [
    ([40, 36, 30], [8, 6, 5], [1, 0, 0], np.float64, 1e-10),
    ([24, 20, 18, 16], [5, 4, 4, 3], [0, 1, 0, 1], np.float64, 1e-10),
    ([96, 64, 80], [12, 10, 8], [1, 1, 0], np.float32, 1e-4),
    ([256, 64, 96], [16, 12, 8], [0, 0, 0], np.float32, 1e-4),
    ([256, 40, 60], [16, 8, 6], [1, 0, 1], np.float32, 1e-4),  # mode 0 on the one-pass ALS kernel
])
def test_two_ranks_one_gpu_host_collectives(dims, ranks, kinds, dtype, tol):
    """N = 2 on the one GPU: both ranks share cuda:0 and exchange through the
    host-staged backend (gloo).  The sharded schedule — per-mode Gram
    allreduce, per-iteration ALS YR/GR allreduce, last-mode all-gather — must
    reproduce the single-process st-HOSVD."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    procs = [mpc.Process(target=_host_comm_worker, args=(r, 2, port, dims, ranks, kinds, dtype, q))
             for r in range(2)]
    for p in procs:
        p.start()
    g, gr, fd, comm_ms = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert abs(g - gr) / gr <= tol
    assert fd <= (1e-8 if dtype == np.float64 else 1e-3)
    assert comm_ms > 0.0


def _schedule_worker(rank, world, port, dims, ranks, kinds, out):
    import os
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2010_10131_b200 import atucker
    from paper_2010_10131_b200.dist import init_host_comm_from_torch, shard_range
    from paper_2010_10131_b200.errors import RankExceedsDim
    from paper_2010_10131_b200.selector import SolverKind, Strategy

    ctx = atucker.Context(0)
    init_host_comm_from_torch(ctx)
    lo, hi = shard_range(dims[-1], rank, world)
    slab = list(dims[:-1]) + [hi - lo]
    xl = atucker.DeviceTensor.uniform(slab, 3, np.float32, ctx=ctx, offset=lo * int(np.prod(dims[:-1])))
    strat = Strategy.manual([SolverKind(k) for k in kinds])
    ctx.comm_stats(reset=True)
    res = atucker.sthosvd(xl, ranks, strat, atucker.AlsOptions(num_iters=3), ctx=ctx, global_dims=dims)
    st = ctx.comm_stats()
    # a rank above the global last dimension fails on every rank alike (no hang)
    bad = list(ranks[:-1]) + [dims[-1] + 1]
    try:
        atucker.sthosvd(xl, bad, strat, ctx=ctx, global_dims=dims)
        failed = False
    except RankExceedsDim:
        failed = True
    out.put((rank, st, list(res.decomposition.core.dims), failed))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dims,ranks,kinds", [
    ([256, 256, 256], [16, 16, 16], [0, 0, 0]),  # C5-shaped at 1/512 of the size
    ([96, 40, 33], [12, 8, 17], [0, 1, 0]),      # uneven slabs 16 / 17 and R_N = 17 > the smaller slab
])
def test_sharded_schedule_collectives(dims, ranks, kinds):
    """SURVEY §8(e) schedule, counted on the host-staged backend (2 ranks on the one GPU):
    one sizes exchange, ONE packed-triangle Gram allreduce per sharded EIG mode
    (I(I+1)/2 doubles), two allreduces (YR, GR) per sharded ALS iteration, and the
    last-mode all-gather (one broadcast per rank) — and nothing else."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    procs = [mpc.Process(target=_schedule_worker, args=(r, 2, port, dims, ranks, kinds, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = len(dims)
    ar_calls, ar_bytes, work = 1, 2 * 8, list(dims)
    for m in range(n - 1):
        i, r = work[m], ranks[m]
        if kinds[m] == 0:
            ar_calls += 1
            ar_bytes += i * (i + 1) // 2 * 8
        else:
            ar_calls += 2 * 3
            ar_bytes += 3 * (i * r + r * r) * 8
        work[m] = r
    gather_bytes = int(np.prod(work)) * 4  # the shrunk tensor before the last mode, fp32
    for rank, st, shape, failed in got:
        assert shape == list(ranks)
        assert failed
        assert st["allreduce_calls"] == ar_calls, st
        assert st["allreduce_bytes"] == ar_bytes, st
        assert st["gather_calls"] == 2, st
        assert st["gather_bytes"] == gather_bytes, st


def _sweep_worker(rank, world, port, cases, out):
    import os
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2010_10131_b200 import atucker
    from paper_2010_10131_b200.dist import init_host_comm_from_torch, shard_range
    from test_gpu_sweep import _PerMode

    ctx = atucker.Context(0)
    init_host_comm_from_torch(ctx)
    plain = atucker.Context(0) if rank == 0 else None
    if plain is not None:
        plain.set_option("als_gram", 0)  # the sharded run iterates over Y (the Gram route is single-GPU)
    for idx, (dims, ranks, kinds, dtype) in enumerate(cases):
        x = np.asfortranarray(np.random.default_rng(idx).standard_normal(dims).astype(dtype))
        lo, hi = shard_range(dims[-1], rank, world)
        xl = atucker.DeviceTensor.from_numpy(np.asfortranarray(x[..., lo:hi]), ctx=ctx)
        opts = atucker.AlsOptions(seed=idx)
        res = atucker.sthosvd(xl, ranks, _PerMode(kinds), opts, ctx=ctx, global_dims=dims)
        xl.free()
        if rank == 0:
            ref = atucker.sthosvd(x, ranks, _PerMode(kinds), opts, ctx=plain)
            core = np.asarray(res.decomposition.core.to_numpy(), dtype=np.float64)
            g = np.linalg.norm(core)
            gr = np.linalg.norm(np.asarray(ref.decomposition.core, dtype=np.float64))
            # the reconstruction error is basis-free: factors of rank-deficient modes (r > rank of
            # the Gram) hold an arbitrary null-space basis in both runs
            dec = atucker.TuckerDecomposition(core.astype(x.dtype), res.decomposition.factors, tuple(dims))
            e = atucker.relative_error(x, dec, ctx=plain)
            er = atucker.relative_error(x, ref.decomposition, ctx=plain)
            out.put((idx, g, gr, abs(e - er)))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_sweep_three_ranks():
    """World size 3 on the one GPU (host-staged collectives, uneven last-mode slabs): the seeded
    sweep's small cases (tests/test_gpu_sweep.py) through the sharded schedule reproduce the
    single-process st-HOSVD: core norm and relative reconstruction error to 1e-10 (fp64) / 1e-4
    (fp32; fixed-order reductions in a different grouping)."""
    import socket

    import torch.multiprocessing as mp

    from test_gpu_sweep import _case

    cases = []
    for s in range(400):
        dims, ranks, kinds, dtype = _case(s)
        if dims[-1] >= 3 and len(cases) < 40:
            cases.append((dims, ranks, kinds, dtype))
    for s in range(16):  # fp32 up to 40M elements: the tensor-core paths, sharded
        dims, ranks, kinds, dtype = _case(s, True)
        if dims[-1] >= 3 and len(cases) < 48:
            cases.append((dims, ranks, kinds, dtype))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mpc = mp.get_context("spawn")
    q = mpc.Queue()
    procs = [mpc.Process(target=_sweep_worker, args=(r, 3, port, cases, q)) for r in range(3)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in cases]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for idx, g, gr, de in got:
        dims, ranks, kinds, dtype = cases[idx]
        tol = 1e-10 if dtype == np.float64 else 1e-4
        assert abs(g - gr) <= tol * gr, (cases[idx], g, gr)
        assert de <= tol, (cases[idx], de)
