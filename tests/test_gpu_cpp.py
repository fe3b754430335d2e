"""The C++ drop-in header (include/atucker_b200.hpp) compiled against the
C ABI and run on the GPU: the reference's calling convention end to end."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _build(tmp_path):
    exe = tmp_path / "test_cpp_dropin"
    lib = ROOT / "paper_2010_10131_b200"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT / 'include'}", str(ROOT / "tests/cpp/test_cpp_dropin.cpp"),
                    f"-L{lib}", "-l:libatk_cuda.so", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    return exe


def test_cpp_dropin_compiles(tmp_path):
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_cpp_dropin_runs(tmp_path):
    out = subprocess.run([str(_build(tmp_path)), str(ROOT / "tests" / "golden"), str(tmp_path)],
                         capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.count("PASS") == 5
