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
