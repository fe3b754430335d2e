""".dten / .tucker formats (tensor_io.hpp:15-99, tucker_io.hpp:20-74) on CPU.

tests/golden/ref_*.dten were written by the reference's OWN write_dten
(oracle/ref_dten.cpp compiled against /root/reference/proj/include,
`make -C oracle dten-goldens`).  The host mirror must read them and write
byte-identical files; the engine's header parser (atk_dten_info, host code in
libatk_cuda.so) must agree; malformed files raise IoFailure with read_dten's
messages.  The device streaming path is tests/test_gpu_tensor_io.py."""
import json
import struct
from pathlib import Path

import numpy as np
import pytest

from paper_2010_10131_b200 import tensor_io as tio
from paper_2010_10131_b200.errors import IoFailure

G = Path(__file__).parent / "golden"
GOLDENS = sorted(G.glob("ref_*.dten"))


def test_goldens_exist():
    assert {p.name for p in GOLDENS} >= {"ref_normal_4x3x5_seed7.dten", "ref_vec5.dten", "ref_matrix_3x2.dten",
                                          "ref_uniform_6x5x4x3_seed11.dten"}


@pytest.mark.parametrize("path", GOLDENS, ids=lambda p: p.name)
def test_host_roundtrip_is_byte_identical(path, tmp_path):
    x = tio.read_dten(path)
    out = tmp_path / "x.dten"
    tio.write_dten(out, x)
    assert out.read_bytes() == path.read_bytes()
    assert tio.dten_info(path) == x.shape


def test_golden_values_are_the_reference_generators(oracle):
    x = tio.read_dten(G / "ref_normal_4x3x5_seed7.dten")
    np.testing.assert_array_equal(x, oracle.random_tensor([4, 3, 5], 7, "normal"))
    u = tio.read_dten(G / "ref_uniform_6x5x4x3_seed11.dten")
    np.testing.assert_array_equal(u, oracle.random_tensor([6, 5, 4, 3], 11, "uniform01"))
    np.testing.assert_array_equal(tio.read_dten(G / "ref_vec5.dten"), [1, 2, 3, 4, 5])
    m = tio.read_dten_matrix(G / "ref_matrix_3x2.dten")
    np.testing.assert_array_equal(m, np.array([[1.5, 4.0], [-2.0, -8.5], [0.25, 16.0]]))
    with pytest.raises(IoFailure, match="expected an order-2"):
        tio.read_dten_matrix(G / "ref_vec5.dten")


def _bad_files(tmp_path):
    good = (G / "ref_normal_4x3x5_seed7.dten").read_bytes()
    hdr = lambda v, n, dims: b"DTEN" + struct.pack("<II", v, n) + struct.pack(f"<{len(dims)}Q", *dims)
    return {
        "bad magic": b"DTEM" + good[4:],
        "unsupported .dten version 2": hdr(2, 3, (4, 3, 5)) + good[28:],
        "truncated or empty header": hdr(1, 0, ()),
        "truncated dims block": hdr(1, 3, (4, 3)),
        "zero dimension": hdr(1, 3, (4, 0, 5)),
        "implausibly large": hdr(1, 2, (1 << 30, 1 << 20)),
        "truncated payload": good[:-8],
    }


def test_malformed_files_raise_iofailure(tmp_path):
    for msg, blob in _bad_files(tmp_path).items():
        p = tmp_path / "bad.dten"
        p.write_bytes(blob)
        if msg != "truncated payload":  # the engine parses headers only
            with pytest.raises(IoFailure, match=msg):
                tio.dten_info(p)
        with pytest.raises(IoFailure, match=msg):
            tio.read_dten(p)
    with pytest.raises(IoFailure, match="cannot open"):
        tio.read_dten(tmp_path / "missing.dten")
    with pytest.raises(IoFailure, match="cannot open"):
        tio.dten_info(tmp_path / "missing.dten")


def test_tucker_directory_roundtrip(tmp_path, oracle):
    from paper_2010_10131_b200.atucker import TuckerDecomposition

    x = oracle.random_tensor([9, 8, 7], 3, "normal")
    ref = oracle.sthosvd(x, [4, 3, 2])
    t = TuckerDecomposition(ref.core, ref.factors, (9, 8, 7))
    tio.save_tucker(tmp_path / "out.tucker", t, [], "eig", 5)
    for f in ["core.dten", "factor_1.dten", "factor_2.dten", "factor_3.dten", "meta.json"]:
        assert (tmp_path / "out.tucker" / f).exists()
    meta = json.loads((tmp_path / "out.tucker" / "meta.json").read_text())
    assert meta == {"original_dims": [9, 8, 7], "ranks": [4, 3, 2], "reports": [], "schema_version": 1,
                    "seed": 5, "strategy": "eig"}
    back = tio.load_tucker(tmp_path / "out.tucker")
    np.testing.assert_array_equal(back.core, ref.core)
    for a, b in zip(back.factors, ref.factors):
        np.testing.assert_array_equal(a, b)
    assert back.original_dims == (9, 8, 7)
    (tmp_path / "out.tucker" / "factor_2.dten").write_bytes((tmp_path / "out.tucker" / "factor_3.dten").read_bytes())
    with pytest.raises(IoFailure, match="factor 2 does not match"):
        tio.load_tucker(tmp_path / "out.tucker")
    with pytest.raises(IoFailure, match="not a .tucker directory"):
        tio.load_tucker(tmp_path / "nope")
