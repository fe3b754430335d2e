"""The C ABI surface (CPU-only checks: load + exports, no compute).

Every function declared in include/atk.h must be exported by
libatk_cuda.so and bound by paper_2010_10131_b200/_lib.py; without a GPU the
library must fail loudly (ATK_CUDA_ERROR), never fall back to the CPU."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared():
    src = (ROOT / "include" / "atk.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(atk_[a-z0-9_]+)\s*\(", src)) - {"atk_selector_fn"})


def test_header_declares_the_hot_path():
    names = declared()
    for must in ["atk_sthosvd", "atk_gram", "atk_ttm", "atk_ttt", "atk_sym_eig_top_r", "atk_eig_mode",
                 "atk_als_mode", "atk_als_iterate", "atk_svd_mode", "atk_thin_qr", "atk_spd_solve",
                 "atk_reconstruct", "atk_relative_error", "atk_comm_init"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2010_10131_b200 import _lib

    lib = _lib.load()
    missing = [n for n in declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared()) == set(_lib.exported_symbols())


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(ROOT / "paper_2010_10131_b200" / "libatk_cuda.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2010_10131_b200 import _lib

    lib = _lib.load()
    h = C.c_void_p()
    assert lib.atk_ctx_create(0, C.byref(h)) == 20  # ATK_CUDA_ERROR
    from paper_2010_10131_b200 import atucker
    from paper_2010_10131_b200.errors import CudaError

    with pytest.raises(CudaError):
        atucker.Context(0)


def test_status_codes_match_oracle():
    """atk_status (atk.h) and the oracle's Status enum share one numbering."""
    src = (ROOT / "oracle" / "atk_oracle.cpp").read_text()
    hdr = (ROOT / "include" / "atk.h").read_text()
    pairs = {"E_ERROR": "ATK_ERROR", "E_NOT_SPD": "ATK_NOT_SPD", "E_RANK_DEFICIENT": "ATK_RANK_DEFICIENT",
             "E_ZERO_NORM_INPUT": "ATK_ZERO_NORM_INPUT", "E_MODE_OUT_OF_RANGE": "ATK_MODE_OUT_OF_RANGE"}
    for o, a in pairs.items():
        vo = re.search(rf"{o} = (\d+)", src).group(1)
        va = re.search(rf"{a} = (\d+)", hdr).group(1)
        assert vo == va
