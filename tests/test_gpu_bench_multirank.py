"""bench.py's N > 1 path (torchrun, one process per rank, max-over-ranks
timing, rank-0 JSON line) exercised on the one test GPU: ATK_BENCH_SHARE_GPU=1
puts both ranks on cuda:0 with host-staged collectives (NCCL refuses two ranks
on one device).  Functional only: a shared GPU gives no scaling number."""
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def test_bench_two_ranks_shared_gpu():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, ATK_BENCH_SHARE_GPU="1")
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
                          "--gpus", "2", "--steps", "2", "--warmup", "3", "--config", "c4"],
                         capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 prints the one line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["ms_per_step"] > 0
    assert d["config"]["parallelism"] == "shard last mode x2"
    assert all(st["comm_ms"] > 0 for st in d["stages"][:-1])  # one Gram allreduce per sharded mode
    assert d["stages"][-1]["comm_ms"] == 0  # the last mode runs on the gathered tensor: no allreduce
    # e2e at N > 1: each rank's slab from pinned host memory through the public sthosvd
    assert d["e2e"]["value"] > 0 and d["e2e"]["h2d_bytes_per_step"] == 4 * 48 ** 5
