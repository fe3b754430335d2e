"""The engine's .dten streaming (csrc/dten_io.cu) on the GPU.

Files written by the reference's own write_dten (tests/golden/ref_*.dten) must
land in HBM exactly (f64) or rounded once (f32); device tensors must come back
as byte-identical files; payloads larger than one 64 MB pinned chunk exercise
the double buffering; and a file-to-file st-HOSVD (read -> sthosvd ->
save_tucker -> load_tucker -> relative_error) matches the CPU oracle."""
from pathlib import Path

import numpy as np
import pytest

from paper_2010_10131_b200 import tensor_io as tio
from paper_2010_10131_b200.errors import IoFailure

pytestmark = pytest.mark.gpu
G = Path(__file__).parent / "golden"


@pytest.mark.parametrize("name", ["ref_normal_4x3x5_seed7.dten", "ref_uniform_6x5x4x3_seed11.dten",
                                  "ref_vec5.dten", "ref_matrix_3x2.dten"])
def test_read_goldens_to_device_and_write_back(ctx, name, tmp_path):
    host = tio.read_dten(G / name)
    d64 = tio.read_dten_device(G / name, np.float64, ctx=ctx)
    np.testing.assert_array_equal(d64.to_numpy(), host)
    d32 = tio.read_dten_device(G / name, np.float32, ctx=ctx)
    np.testing.assert_array_equal(d32.to_numpy(), host.astype(np.float32))
    tio.write_dten(tmp_path / "back.dten", d64)
    assert (tmp_path / "back.dten").read_bytes() == (G / name).read_bytes()
    tio.write_dten(tmp_path / "back32.dten", d32)
    np.testing.assert_array_equal(tio.read_dten(tmp_path / "back32.dten"), host.astype(np.float32).astype(np.float64))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_multi_chunk_streaming(ctx, dtype, tmp_path):
    from paper_2010_10131_b200 import atucker

    dims = (160, 250, 430)  # 17.2 M elements: 137 MB of f64 payload = 3 chunks
    x = atucker.DeviceTensor.uniform(list(dims), 9, dtype, ctx=ctx)
    p = tmp_path / "big.dten"
    tio.write_dten(p, x)
    assert p.stat().st_size == 4 + 4 + 4 + 3 * 8 + 8 * int(np.prod(dims))
    want = x.to_numpy().astype(np.float64)
    np.testing.assert_array_equal(tio.read_dten(p), want)
    y = tio.read_dten_device(p, dtype, ctx=ctx)
    np.testing.assert_array_equal(y.to_numpy(), x.to_numpy())
    raw = p.read_bytes()
    p.write_bytes(raw[:-12])
    with pytest.raises(IoFailure, match="truncated payload"):
        tio.read_dten_device(p, dtype, ctx=ctx)


def test_file_to_file_sthosvd_matches_oracle(ctx, oracle, tmp_path):
    from paper_2010_10131_b200 import atucker
    from paper_2010_10131_b200.selector import Strategy

    x = oracle.random_tensor([30, 26, 22], 4, "normal")
    src = tmp_path / "in.dten"
    tio.write_dten(src, x)
    xd = tio.read_dten_device(src, np.float64, ctx=ctx)
    res = atucker.sthosvd(xd, [6, 5, 4], Strategy.fixed_eig(), ctx=ctx)
    tio.save_tucker(tmp_path / "out.tucker", res.decomposition, res.reports, "eig", 0)
    back = tio.load_tucker(tmp_path / "out.tucker")
    ref = oracle.sthosvd(x, [6, 5, 4])
    g, gr = np.linalg.norm(back.core), np.linalg.norm(ref.core)
    assert abs(g - gr) / gr <= 1e-10
    e = atucker.relative_error(x, back, ctx=ctx)
    er = oracle.relative_error(x, ref.core, ref.factors)
    assert abs(e - er) <= 1e-10
    import json

    meta = json.loads((tmp_path / "out.tucker" / "meta.json").read_text())
    assert [r["mode"] for r in meta["reports"]] == [1, 2, 3]
    assert meta["reports"][0]["solver"] == "eig" and meta["reports"][0]["dims_after"] == [6, 26, 22]
