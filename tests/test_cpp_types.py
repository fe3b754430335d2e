"""The C++ drop-in against the reference's own types (CPU, no GPU needed).

include/atucker_b200.hpp consumes the reference's Eigen-free headers when they
are on the include path (atucker::DenseTensor / DenseMatrix, the errors.hpp
exception hierarchy, atucker::SolverKind, selector::predict).  Built both
ways and run: status -> exception mapping, the selector-hook trampoline with
the reference's decide signature, the cost model's num_iters, the Adaptive
tree.  The GPU drop-in test (tests/cpp/test_cpp_dropin.cpp) is also compiled
and linked against the reference headers here.
"""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF_INC = Path("/root/reference/proj/include")
LIB = ROOT / "paper_2010_10131_b200"


def _build(src, exe, extra):
    subprocess.run(["g++", "-std=c++20", "-O1", "-Wall", f"-I{ROOT / 'include'}", *extra, str(src),
                    f"-L{LIB}", "-l:libatk_cuda.so", f"-Wl,-rpath,{LIB}", "-o", str(exe)], check=True)
    return exe


@pytest.mark.parametrize("mode", ["reference", "standalone"])
def test_cpp_types(tmp_path, mode):
    if not (LIB / "libatk_cuda.so").exists():
        pytest.skip("libatk_cuda.so not built")
    if mode == "reference":
        if not (REF_INC / "atucker" / "tensor.hpp").exists():
            pytest.skip("reference headers not mounted (GPU box)")
        extra = [f"-I{REF_INC}"]
    else:
        extra = ["-DATUCKER_B200_STANDALONE"]
    exe = _build(ROOT / "tests/cpp/test_cpp_types.cpp", tmp_path / "t", extra)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("PASS") == 6, out.stdout
    assert ("PASS reference types" in out.stdout) == (mode == "reference")


def test_cpp_dropin_links_against_reference_types(tmp_path):
    if not (LIB / "libatk_cuda.so").exists() or not (REF_INC / "atucker" / "tensor.hpp").exists():
        pytest.skip("needs the built library and the reference headers")
    assert _build(ROOT / "tests/cpp/test_cpp_dropin.cpp", tmp_path / "d", [f"-I{REF_INC}"]).exists()
